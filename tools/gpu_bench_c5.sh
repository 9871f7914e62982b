timeout 900 python bench.py --workload c5 --steps 5 --warmup 3 > gpurun_out/c5_bench.json 2> gpurun_out/c5_bench.err; echo "c5 rc=$?"
python - <<'PY'
import json
d = json.loads(open("gpurun_out/c5_bench.json").read().strip().splitlines()[-1])
print("value %.4g ms %.2f e2e %.4g frac %.3f" % (d["value"], d["ms_per_step"], d["e2e"]["value"], d["roofline"]["frac"]), d["clocks"], d.get("parity"), d.get("cpu_baseline", {}).get("value"))
PY
