# N>1 bench path (torchrun, one process per rank) with every rank on cuda:0 (test hook) —
# exercises DistributedPipeline + IPC rings + the GPU-sharing policy on a 1-GPU box
export PPLL_BENCH_SHARE_GPU=1
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29711 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/mr_vit2.json 2> gpurun_out/mr_vit2.err; echo "vit_s N=2 rc=$?"
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29712 bench.py --gpus 4 --workload resnet32 --steps 10 --warmup 3 > gpurun_out/mr_res4.json 2> gpurun_out/mr_res4.err; echo "resnet32 N=4 rc=$?"
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29713 bench.py --impl reference --gpus 2 --steps 3 --warmup 1 > gpurun_out/mr_ref2.json 2> gpurun_out/mr_ref2.err; echo "reference N=2 rc=$?"
