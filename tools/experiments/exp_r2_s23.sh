# S23 bench step (2048 sampled sources): lane width x pipelines (auto: W = 4, 1 pipeline)
nvidia-smi --query-gpu=memory.total,memory.used --format=csv
for cfg in "0 0" "4 2" "2 0" "2 2" "2 3"; do set -- $cfg
  echo -n "S23 W=$1 streams=$2: "; timeout 600 python tools/prof_batch.py --scale 23 --sources 2048 --lane-words $1 --streams $2 --repeat 2 --no-profile 2>&1 | tail -1 | cut -c1-100
done
