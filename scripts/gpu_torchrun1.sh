# the multi-GPU launch path (torchrun, NCCL, max-over-ranks timing) at world size 1 on the box
mkdir -p gpurun_out/trun
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 5 --warmup 3 > gpurun_out/trun/ours.json 2> gpurun_out/trun/ours.err
echo "ours rc=$?"; head -c 600 gpurun_out/trun/ours.json; echo
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 1 --steps 5 --warmup 3 > gpurun_out/trun/ref.json 2> gpurun_out/trun/ref.err
echo "ref rc=$?"; head -c 400 gpurun_out/trun/ref.json; echo
timeout 600 python bench.py --gpus 1 --steps 5 --warmup 3 --workload ml20m > gpurun_out/trun/ml20m.json 2> gpurun_out/trun/ml20m.err
echo "ml20m rc=$?"; head -c 300 gpurun_out/trun/ml20m.json; echo
tail -3 gpurun_out/trun/ours.err
