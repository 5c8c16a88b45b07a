# round 2, multi-GPU call m: final-tree SFT bench (defaults), BASELINE configs[3]/[4] at N (Llama-3-8B 32K, Qwen2.5-14B 64K FIXED) + fetch CTA budget A/B
set -x
N=$(nvidia-smi -L | wc -l)
D=gpurun_out/r02m_n$N
mkdir -p $D
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29530 bench.py --gpus $N > $D/bench_final.json 2> $D/bench_final.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29531 bench_p2p.py --sizes 16M,32M --variants tma:96,tma:128,tma:148 --out $D/p2p_fetch_ctas.md > $D/p2p_fetch_ctas.jsonl 2> $D/p2p.err
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29532 bench.py --gpus $N --steps 6 --warmup 3 --model llama-3-8b --no-cpu-baseline --no-e2e > $D/bench_llama8b.json 2> $D/bench_llama8b.err
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $N --steps 4 --warmup 3 --model qwen2.5-14b --cap 65536 --push-mode fixed --no-cpu-baseline --no-e2e > $D/bench_qwen14b_fixed_64k.json 2> $D/bench_qwen14b.err
cat $D/p2p_fetch_ctas.md; grep -h '^{' $D/bench_*.json | cut -c1-300
