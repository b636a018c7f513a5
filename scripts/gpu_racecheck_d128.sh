# compute-sanitizer racecheck on the d_h = 128 tensor-core kernels (small shapes)
mkdir -p gpurun_out/race
for c in tchsmall tcgsmall; do
  timeout 1200 compute-sanitizer --tool racecheck --print-limit 5 python scripts/sanitize_case.py $c > gpurun_out/race/racecheck_$c.log 2>&1
  echo "racecheck $c: $(grep -E 'RACECHECK SUMMARY|ERROR SUMMARY|parity ok' gpurun_out/race/racecheck_$c.log | tr '\n' ' ')"
done
