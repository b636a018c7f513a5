# compute-sanitizer on the round-2 tensor-core kernels (and the rest), multi-unit shapes, values checked
mkdir -p gpurun_out/san
for c in tcf64 tcflong tcfmerge tcb64 tcbpair tcblong tc; do
  for tool in memcheck synccheck; do
    timeout 600 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_case.py $c > gpurun_out/san/${tool}_$c.log 2>&1
    echo "$tool $c: $(grep -E 'ERROR SUMMARY|parity ok' gpurun_out/san/${tool}_$c.log | tr '\n' ' ')"
  done
done
for c in tcf64 tcfmerge tcbpair; do
  timeout 900 compute-sanitizer --tool racecheck --print-limit 5 python scripts/sanitize_case.py $c > gpurun_out/san/racecheck_$c.log 2>&1
  echo "racecheck $c: $(grep -E 'RACECHECK SUMMARY|ERROR SUMMARY|parity ok' gpurun_out/san/racecheck_$c.log | tr '\n' ' ')"
done
