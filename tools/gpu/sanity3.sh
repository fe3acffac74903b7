for tool in memcheck racecheck synccheck initcheck; do
  echo "== $tool"; timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 python tools/gpu/sanitize.py 2>&1 | tail -3
done
