for w in c1 c3 c4; do
timeout 900 python bench.py --workload $w --steps 3 --warmup 3 > gpurun_out/${w}_bench.json 2> gpurun_out/${w}_bench.err; echo "$w rc=$?"
done
python - <<'PY'
import json
for w in ("c1", "c3", "c4"):
    try:
        d = json.loads(open(f"gpurun_out/{w}_bench.json").read().strip().splitlines()[-1])
    except Exception as e:
        print(w, "no line", e); continue
    print(w, "value %.4g ms %.2f e2e %.4g frac %.3f" % (d["value"], d["ms_per_step"], d["e2e"]["value"], d["roofline"]["frac"] or 0), "cpu %.3g" % (d.get("cpu_baseline") or {}).get("value", 0), d.get("parity"))
PY
