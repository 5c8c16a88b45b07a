# round 2, multi-GPU call j: new fetch pipeline P2P, SFT bench RED vs SLOT push (same box, back to back)
set -x
N=$(nvidia-smi -L | wc -l)
D=gpurun_out/r02j_n$N
mkdir -p $D
python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29521 bench_p2p.py --sizes 4M,16M,32M,64M,256M --out $D/p2p.md > $D/p2p.jsonl 2> $D/p2p.err
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29522 bench.py --gpus $N --steps 20 --warmup 5 --push-mode slot --no-cpu-baseline > $D/bench_slot.json 2> $D/bench_slot.err
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29523 bench.py --gpus $N --steps 20 --warmup 5 --push-mode red --no-cpu-baseline > $D/bench_red.json 2> $D/bench_red.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29524 bench.py --gpus $N --impl reference --steps 20 --warmup 5 > $D/bench_ref.json 2> $D/bench_ref.err
cat $D/p2p.md; grep '^{' $D/bench_slot.json | head -c 400; echo; grep '^{' $D/bench_red.json | head -c 400
