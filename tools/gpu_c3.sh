timeout 900 python bench.py --workload c3 --steps 3 --warmup 3 > gpurun_out/c3_bench.json 2> gpurun_out/c3_bench.err; echo "c3 rc=$?"; tail -3 gpurun_out/c3_bench.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/c3_bench.json").read().strip().splitlines()[-1])
print("value %.4g ms %.2f e2e %.4g frac %.3f" % (d["value"], d["ms_per_step"], d["e2e"]["value"], d["roofline"]["frac"] or 0), d.get("parity"), d["pool_roofline"]["pool_ms_per_step"])
PY
