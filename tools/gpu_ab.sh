# Parity tests, per-level contraction timings, and a short bench.
python __graft_entry__.py
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.log | grep -v "^$"
timeout 300 python tools/bench_level.py c2 2>&1 | tail -3
timeout 300 python tools/bench_level.py c4 1:16384 2:64360 3:14796 2>&1 | tail -3
for i in 1 2; do
  timeout 300 python bench.py --steps 30 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench', d['ms_per_step'], d['e2e']['value'], d['roofline'])"
done
