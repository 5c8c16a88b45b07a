# round 2, multi-GPU call (run with gpurun --gpus N; N from nvidia-smi): P2P engines vs NCCL, NVLink counters,
# multi-process protocol tests, SFT bench with the FSDP arm
set -x
N=$(nvidia-smi -L | wc -l)
D=gpurun_out/r02e_n$N
mkdir -p $D
python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench_p2p.py --sizes 1M,4M,16M,32M,64M,256M --out $D/p2p.md > $D/p2p.jsonl 2> $D/p2p.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29512 bench_p2p.py --sizes 4M,16M,64M --sync --reps 10 --out $D/p2p_sync.md > $D/p2p_sync.jsonl 2> $D/p2p_sync.err
timeout 300 python tools/nvlink_probe.py --gpus $N --mb 16 > $D/nvlink_probe.jsonl 2>&1
timeout 900 python -m pytest tests/test_engine_multigpu.py tests/test_worker_multigpu.py tests/test_engine_local_group_gpu.py tests/test_fabric_gpu.py -q --timeout 600 -p no:cacheprovider > $D/tests.log 2>&1
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus $N --steps 10 --warmup 3 --no-cpu-baseline > $D/bench.json 2> $D/bench.err
timeout 600 ncu --devices 0 --metrics gpu__time_duration.sum,nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:"fetch|push_bulk|push_red" --csv --log-file $D/ncu_nvlink.csv python tools/nvlink_probe.py --gpus $N --mb 16 --reps 2 > $D/ncu_run.log 2>&1
ODC_DEVICES=$(seq -s, 0 $((N-1))) timeout 300 tests/refsuite/_build/ref_primitives_tests > $D/refsuite_primitives_multigpu.log 2>&1
tail -3 $D/tests.log; tail -2 $D/refsuite_primitives_multigpu.log; cat $D/bench.json
