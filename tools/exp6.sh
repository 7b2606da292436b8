for part in base bidx flag overlap; do
  echo "== $part"
  SANITIZE_PART=$part timeout 300 compute-sanitizer --tool racecheck python tools/sanitize.py 2>&1 | grep -E "Race reported|at .*tagg_ptx|SUMMARY" | head -12
done
