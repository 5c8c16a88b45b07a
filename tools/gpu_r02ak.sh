# round 2, call ak (4 GPUs): final tree: multi-GPU protocol tests, the N=4 SFT bench (driver window) with the
# same-box FSDP arm, and the reference arm at N=4 (rank 0 only)
set -x
N=$(nvidia-smi -L | wc -l)
D=gpurun_out/r02ak_n$N
mkdir -p $D
timeout 1200 python -m pytest tests/test_engine_multigpu.py tests/test_worker_multigpu.py tests/test_engine_local_group_gpu.py tests/test_fabric_gpu.py tests/test_world8_step_gpu.py -q --timeout 900 -p no:cacheprovider > $D/tests.log 2>&1
timeout 1800 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29613 bench.py --gpus $N > $D/bench.json 2> $D/bench.err
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29614 bench.py --impl reference --gpus $N > $D/bench_ref.json 2> $D/bench_ref.err
tail -n 2 $D/tests.log; grep '^{' $D/bench.json | cut -c1-300; grep '^{' $D/bench_ref.json | cut -c1-300
