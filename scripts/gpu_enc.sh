# Encoder step parity (tests/test_encoder_gpu.py) + the op's parity tests
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_encoder_gpu.py -q -p no:cacheprovider -x --durations=5 > gpurun_out/pytest_enc.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_enc.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_reference_api_gpu.py -q -p no:cacheprovider -x > gpurun_out/pytest_op.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_op.log
tail -30 gpurun_out/pytest_enc.log; tail -3 gpurun_out/pytest_op.log
