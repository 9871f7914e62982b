# A/B of per-level contraction timings: current tree vs _ab_old (a worktree of the previous commit).
for i in 1 2 3; do
  echo new; FC_BENCH_REPS=30 timeout 300 python tools/bench_level.py c2 2>&1 | tail -3
  echo old; (cd _ab_old && FC_BENCH_REPS=30 timeout 300 python tools/bench_level.py c2 2>&1 | tail -3)
done
