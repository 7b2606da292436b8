for part in overlap base; do
  echo "== $part"
  SANITIZE_PART=$part timeout 300 compute-sanitizer --tool racecheck python tools/sanitize.py 2>&1 | grep -E "cp_async|SUMMARY" | head -4
done
timeout 60 compute-sanitizer --tool racecheck ./tools/micro/alloc_race 3 2>&1 | tail -8
