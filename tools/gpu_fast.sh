#!/bin/bash
# Fast modes (1e-2 tolerance) and the C5 scaling workload; torchrun (world size 1) launch of both arms.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out/fast
O=gpurun_out/fast
timeout 600 python bench.py --precision tf32 --steps 30 --warmup 5 --no-cpu-baseline > $O/alexnet_tf32.json 2> $O/alexnet_tf32.err
timeout 600 python bench.py --precision bf16 --steps 30 --warmup 5 --no-cpu-baseline > $O/alexnet_bf16.json 2> $O/alexnet_bf16.err
timeout 600 python bench.py --workload vgg16 --precision tf32 --steps 10 --warmup 3 --no-cpu-baseline > $O/vgg_tf32.json 2> $O/vgg_tf32.err
timeout 600 python bench.py --workload vgg16 --precision bf16 --steps 10 --warmup 3 --no-cpu-baseline > $O/vgg_bf16.json 2> $O/vgg_bf16.err
timeout 600 python bench.py --workload scale --steps 10 --warmup 3 --no-cpu-baseline > $O/scale_fp32.json 2> $O/scale_fp32.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu-baseline > $O/torchrun_ours.json 2> $O/torchrun_ours.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29532 bench.py --impl reference --gpus 1 --steps 2 --warmup 1 > $O/torchrun_ref.json 2> $O/torchrun_ref.err
