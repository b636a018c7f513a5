# encoder tests + encoder bench after the colsum change; ncu of tcf / tcb after the splitter fix
mkdir -p gpurun_out/r02n
timeout 600 python -m pytest tests/test_encoder_gpu.py -q -p no:cacheprovider > gpurun_out/r02n/pytest_enc.log 2>&1; echo "rc=$?" >> gpurun_out/r02n/pytest_enc.log
tail -3 gpurun_out/r02n/pytest_enc.log
timeout 600 python bench.py --encoder-only --steps 10 --warmup 3 --no-cpu > gpurun_out/r02n/bench_enc.json 2> gpurun_out/r02n/bench_enc.err
python -c "
import json; d=json.load(open('gpurun_out/r02n/bench_enc.json')); e=d.get('encoder_step', d); print('encoder', e.get('value'), e.get('ms_per_step'), e.get('phases_ms'))" 2>&1 | tail -2
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tcf_kernel -c 2 -o gpurun_out/r02n/prof_tcf -f python bench.py --workload sw_n4096_d64_f32 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/r02n/prof_tcf.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tcb_kernel -c 2 -o gpurun_out/r02n/prof_tcb64 -f python bench.py --workload sw_n4096_d64_bf16 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/r02n/prof_tcb.log 2>&1
ls gpurun_out/r02n
