# full GPU suite + smoke + sanitizer on the d_h = 128 tensor-core kernels
mkdir -p gpurun_out/val
timeout 2400 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/val/pytest_gpu.txt 2>&1
tail -5 gpurun_out/val/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
for c in tch tchlong tcg tcglong; do
  for tool in memcheck synccheck; do
    timeout 600 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_case.py $c > gpurun_out/val/${tool}_$c.log 2>&1
    echo "$tool $c: $(grep -E 'ERROR SUMMARY|parity ok' gpurun_out/val/${tool}_$c.log | tr '\n' ' ')"
  done
done
