# Parity tests + launch list of three c2 encodes (kernel times).
python __graft_entry__.py
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log | grep -v "^$"
timeout 300 python tools/prof_c2.py c2 > gpurun_out/prof_c2_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python tools/prof_c2.py c2 > gpurun_out/ncu_c2.log 2>&1; echo "ncu rc=$?"
for i in 1 2; do
  timeout 300 python bench.py --steps 30 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench', d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'])"
done
