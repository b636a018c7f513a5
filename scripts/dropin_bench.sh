# The reference encoder (compiled unmodified) with and without the B200
# operator under it, ML-1M shape, all host threads: model_forward +
# model_backward seconds per step (tests/cpp/dropin_main.cpp bench mode).
T=$(nproc); B=${1:-64}; R=${2:-3}
mkdir -p gpurun_out
./tests/cpp/_build/dropin_ref /tmp/dref.bin $T bench $B $R | tee gpurun_out/dropin_bench.txt
COTTEN_ADAPTER_DTYPE=f32 ./tests/cpp/_build/dropin_gpu /tmp/dgpu.bin $T bench $B $R | tee -a gpurun_out/dropin_bench.txt
python - <<'PY' | tee -a gpurun_out/dropin_bench.txt
import numpy as np
a = np.fromfile('/tmp/dref.bin'); b = np.fromfile('/tmp/dgpu.bin')
print('parity normwise', float(np.abs(a - b).max() / np.abs(a).max()), 'values', a.size)
PY
