# A/B of the epilogue drain layout (FC_TC_G1) with parity tests for both.
python __graft_entry__.py
FC_TC_G1=1 timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_g1.log 2>&1; echo "pytest g1 rc=$?"; tail -2 gpurun_out/pytest_gpu_g1.log
for g in 0 1; do
  echo "G1=$g"; FC_TC_G1=$g timeout 300 python tools/bench_level.py c2 2>&1 | tail -3
  FC_TC_G1=$g timeout 300 python tools/bench_level.py c4 1:16384 2:64360 3:14796 2>&1 | tail -3
done
