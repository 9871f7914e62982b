# Parity tests with PDL on, then bench A/B of FC_PDL.
python __graft_entry__.py
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
for p in 1 0 1 0; do
  FC_PDL=$p timeout 300 python bench.py --steps 30 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('pdl=$p', d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'])"
done
