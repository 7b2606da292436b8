for part in overlap_sync overlap; do
  echo "== $part"
  SANITIZE_PART=$part timeout 300 compute-sanitizer --tool racecheck python tools/sanitize.py 2>&1 | grep -E "cp_async|SUMMARY" | head -4
done
for m in 2 3; do timeout 60 compute-sanitizer --tool racecheck ./tools/micro/alloc_race $m 2>&1 | tail -4; done
