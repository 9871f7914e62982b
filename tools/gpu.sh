# GPU-box entry points (run through gpurun from the repo root):
#   bash tools/gpu.sh iter         parity suite + per-level contraction timings (c2 both modes, c5 L2)
#   bash tools/gpu.sh shist        s-histogram parity + timing (c2)
#   bash tools/gpu.sh ncu-shist    ncu --set full of the s-histogram search (c2 level 2)
#   bash tools/gpu.sh ncu-c5 [OUT] ncu --set full of the c5 level-2 contraction
#   bash tools/gpu.sh bench        bench lines c5 (headline) and c2, summarised
#   bench-all                      bench lines c1, c3, c4
#   profile                        round evidence: launch lists of the c5 / c2 bench
# Every ncu run follows a plain run of the same command that exited 0.
cmd=${1:-iter}
summary() {
python - "$@" <<'PY'
import json, sys
for w in sys.argv[1:]:
    try:
        d = json.loads(open(f"gpurun_out/{w}_bench.json").read().strip().splitlines()[-1])
    except Exception as e:
        print(w, "no line", e); continue
    print(w, "value %.4g ms/step %.3f e2e %.4g frac %.3f" % (d["value"], d["ms_per_step"], d["e2e"]["value"],
          d["roofline"]["frac"] or 0), "clk", d["clocks"], "cpu", (d.get("cpu_baseline") or {}).get("value"),
          d.get("parity"))
PY
}
case "$cmd" in
iter)
  timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
  FC_BENCH_REPS=5 timeout 300 python tools/bench_level.py c2 2>&1 | tail -3
  FC_MODE=baseline FC_BENCH_REPS=3 timeout 300 python tools/bench_level.py c2 2>&1 | tail -3
  FC_BENCH_REPS=2 timeout 300 python tools/bench_level.py c5 2:65536 2>&1 | tail -1
  ;;
shist)
  timeout 600 python -m pytest tests/test_shist.py -q -x > gpurun_out/pytest_shist.log 2>&1; echo "shist tests rc=$?"; tail -2 gpurun_out/pytest_shist.log
  timeout 300 python tools/time_shist.py c2 2>&1 | tail -4
  ;;
ncu-shist)
  timeout 300 python tools/shist_once.py c2 > gpurun_out/shist_once.log 2>&1 && \
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:tc_scan_kernel -s 1 -c 1 -f \
    -o gpurun_out/tc_real_c2 python tools/shist_once.py c2 > gpurun_out/ncu_real.log 2>&1; echo "ncu rc=$?"
  ;;
ncu-c5)
  out=${2:-tc_scan_c5_full}
  export FC_BENCH_REPS=1
  timeout 300 python tools/bench_level.py c5 2:65536 > gpurun_out/c5_level.txt 2>&1 && \
  timeout 1200 ncu --set full --import-source on --clock-control none -k regex:tc_scan_kernel -c 1 -f \
    -o gpurun_out/$out python tools/bench_level.py c5 2:65536 > gpurun_out/ncu_c5.log 2>&1; echo "ncu rc=$?"
  cat gpurun_out/c5_level.txt
  ;;
bench)
  timeout 900 python bench.py --workload c5 --steps 5 --warmup 3 > gpurun_out/c5_bench.json 2> gpurun_out/c5_bench.err; echo "c5 rc=$?"
  timeout 300 python bench.py --workload c2 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/c2_bench.json 2> gpurun_out/c2_bench.err; echo "c2 rc=$?"
  summary c5 c2
  ;;
bench-all)
  for w in c1 c3 c4; do
    timeout 900 python bench.py --workload $w --steps 3 --warmup 3 > gpurun_out/${w}_bench.json 2> gpurun_out/${w}_bench.err; echo "$w rc=$?"
  done
  summary c1 c3 c4
  ;;
profile)
  timeout 600 python bench.py --workload c5 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/c5_plain.json 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_c5.csv \
    python bench.py --workload c5 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "launches c5 rc=$?"
  timeout 300 python bench.py --workload c2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/c2_plain.json 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_c2.csv \
    python bench.py --workload c2 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "launches c2 rc=$?"
  ;;
*) echo "unknown command $cmd"; exit 2 ;;
esac
