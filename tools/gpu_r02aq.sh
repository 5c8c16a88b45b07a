# round 2, call aq (4 GPUs): BASELINE configs[3] (Llama-3-8B, 32K cap) and configs[4] (Qwen2.5-14B, 64K cap,
# FIXED deterministic push) on the final tree, with the same-box FSDP arm
set -x
N=$(nvidia-smi -L | wc -l)
D=gpurun_out/r02aq_n$N
mkdir -p $D
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29632 bench.py --gpus $N --steps 6 --warmup 3 --model llama-3-8b --no-cpu-baseline --no-e2e > $D/bench_llama8b.json 2> $D/bench_llama8b.err
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29633 bench.py --gpus $N --steps 4 --warmup 3 --model qwen2.5-14b --cap 65536 --push-mode fixed --no-cpu-baseline --no-e2e > $D/bench_qwen14b_fixed_64k.json 2> $D/bench_qwen14b.err
grep '^{' $D/bench_llama8b.json | cut -c1-200; grep '^{' $D/bench_qwen14b_fixed_64k.json | cut -c1-200
