# N>1 bench orchestration on ONE device (FDIRW_BENCH_ONE_DEVICE=1: gloo, P2P over CUDA IPC, both
# ranks on cuda:0): the same code path as the driver's torchrun launch minus NVLink
set -x
python -c "import __graft_entry__ as g; g.build()"
FDIRW_BENCH_ONE_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 20 --warmup 5 \
  > gpurun_out/onedev_n2.log 2> gpurun_out/onedev_n2.err
echo rc=$?
tail -5 gpurun_out/onedev_n2.err
