# Interleaved A/B of an environment switch: gpu_ab_env.sh VAR "A B" [rounds]
var=$1; vals=$2; rounds=${3:-3}
python __graft_entry__.py
for i in $(seq $rounds); do
  for v in $vals; do
    env $var=$v TAG="$var=$v" timeout 300 python tools/step_time.py c2 150 2>&1 | tail -1
  done
done
