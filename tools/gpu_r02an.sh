# round 2, call an (2 GPUs): N=2 SFT bench of the final tree (driver window) with the FSDP arm
set -x
N=$(nvidia-smi -L | wc -l)
D=gpurun_out/r02an_n$N
mkdir -p $D
ODC_BENCH_LOG=1 timeout 1800 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29615 bench.py --gpus $N > $D/bench.json 2> $D/bench.err
grep '^{' $D/bench.json | cut -c1-300; grep "timed steps done" $D/bench.err | head -4
