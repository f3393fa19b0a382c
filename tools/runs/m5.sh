cd $GRAFT_REPO_ROOT
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,nvlrx__bytes.sum,nvltx__bytes.sum"
NCU_MULTI_RANK=1 timeout 600 python tools/ncu_multi.py --world 2 --out gpurun_out/m5_ncu_p2 --metrics "$M" > gpurun_out/m5_ncu_p2.log 2>&1; echo ncu rc=$?
tail -n 3 gpurun_out/m5_ncu_p2.log; for f in gpurun_out/m5_ncu_p2.rank*.log; do echo "== $f"; grep -v "^  " $f | head -12; done
head -c 1500 gpurun_out/m5_ncu_p2.csv
