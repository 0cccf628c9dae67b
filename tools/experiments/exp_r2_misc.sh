# S20 8192 sources (device loop, auto pipelines): batch order, hub split, lane width
for opt in "" "--order 3" "--hub 2048" "--hub 8192" "--lane-words 8" "" "--order 3"; do
  echo -n "[$opt] S20: "; timeout 200 python tools/prof_batch.py --sources 8192 --lane-words 0 --repeat 3 --no-profile $opt | tail -1 | cut -c1-80
done
