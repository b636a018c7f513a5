# BASELINE config #5: the long-sequence sweep (N x d_h x dtype) on one B200;
# one bench line per point into gpurun_out/sweep/, then a table.
mkdir -p gpurun_out/sweep
for n in 512 1024 2048 4096 8192 16384; do for d in 32 64 128; do for dt in f32 bf16; do
  w=sw_n${n}_d${d}_${dt}
  timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/sweep/$w.json 2>gpurun_out/sweep/$w.err
done; done; done
python scripts/sweep_table.py gpurun_out/sweep | tee gpurun_out/sweep/table.md
