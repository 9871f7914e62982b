# headline bench (c5) + c2 line, then the launch list of the c5 bench
timeout 900 python bench.py --workload c5 --steps 5 --warmup 3 > gpurun_out/c5_bench.json 2> gpurun_out/c5_bench.err; echo "c5 rc=$?"
timeout 300 python bench.py --workload c2 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/c2_bench.json 2> gpurun_out/c2_bench.err; echo "c2 rc=$?"
python - <<'PY'
import json
for f in ("c5_bench", "c2_bench"):
    try:
        d = json.loads(open(f"gpurun_out/{f}.json").read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "no line", e); continue
    print(f, "value %.4g" % d["value"], "ms/step %.3f" % d["ms_per_step"], "e2e %.4g" % d["e2e"]["value"],
          "frac %.3f" % d["roofline"]["frac"], "kernel ms %.3f" % d["roofline"]["kernel_ms_per_step"],
          "clk", d["clocks"], "cpu", (d.get("cpu_baseline") or {}).get("value"), d.get("parity"))
PY
