# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_run.py (every kernel family, small graphs)
for tool in memcheck racecheck synccheck; do
  for w in lanes slices; do
    echo "== $tool $w"
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py $w 2>&1 | tail -6
  done
done
