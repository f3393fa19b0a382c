cd $GRAFT_REPO_ROOT
cat > /tmp/k.py <<'PY'
import torch
x = torch.randn(1 << 24, device="cuda"); y = x * 2; torch.cuda.synchronize(); print("ok")
PY
for M in gpu__time_duration.sum "gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum" "nvlrx__bytes.sum,nvltx__bytes.sum" "gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,nvlrx__bytes.sum,nvltx__bytes.sum"; do
  echo "== $M"; timeout 120 ncu --metrics $M -c 1 python /tmp/k.py 2>&1 | grep -E "PROF|pass|replay|ok" | head -5
done
