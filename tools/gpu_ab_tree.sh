# Interleaved step-time A/B: current tree vs _ab_old (a worktree with one change reverted).
for i in 1 2 3; do
  TAG=new timeout 300 python tools/step_time.py c2 150 2>&1 | tail -1
  (cd _ab_old && TAG=old timeout 300 python tools/step_time.py c2 150 2>&1 | tail -1)
done
