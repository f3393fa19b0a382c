cd $GRAFT_REPO_ROOT
for w in 2; do
timeout 400 python tools/ncu_multi.py --world $w --out gpurun_out/m9_ncu_dram_p$w --metrics "gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum" > gpurun_out/m9_dram_p$w.log 2>&1; echo "dram p$w rc=$?"
timeout 400 python tools/ncu_multi.py --world $w --out gpurun_out/m9_ncu_nvl_p$w --metrics "nvlrx__bytes.sum,nvltx__bytes.sum" > gpurun_out/m9_nvl_p$w.log 2>&1; echo "nvl p$w rc=$?"
grep -c "k_" gpurun_out/m9_ncu_dram_p$w.csv gpurun_out/m9_ncu_nvl_p$w.csv
done
