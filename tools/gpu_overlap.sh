# Overlap A/B: parity tests, then bench.py with and without the second stream.
python __graft_entry__.py
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.log | grep -v "^$"
for o in 1 0 1 0; do
  FC_OVERLAP=$o timeout 300 python bench.py --steps 30 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('overlap=$o', d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'])"
done
FC_TRACE=1 FC_REPS=2 timeout 300 python tools/time_encode.py c2 2>&1 | grep -E "it1|phases|level" | head -12
