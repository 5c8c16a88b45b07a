# round 2, call l: attention order A/B (previous build vs lockstep order), attention/engine tests,
# final-tree N=1 bench (both arms) + the ncu launch list of the same bench command
set -x
D=gpurun_out/r02l
mkdir -p $D
(cd _ab/v2 && timeout 300 python attn_bwd_ab.py) > $D/attn_prev_order.jsonl 2>&1
timeout 300 python tools/attn_bwd_ab.py > $D/attn_lockstep.jsonl 2>&1
timeout 900 python -m pytest tests/test_attention_gpu.py tests/test_engine_local_group_gpu.py tests/test_engine_gpu.py -q --timeout 600 -p no:cacheprovider > $D/tests.log 2>&1
timeout 300 python -m pytest tests/test_bench_config_gpu.py -q -k attention --timeout 600 -p no:cacheprovider > $D/tests_attn_big.log 2>&1
timeout 900 python bench.py > $D/bench_n1.json 2> $D/bench_n1.err
timeout 900 python bench.py --impl reference > $D/bench_ref_n1.json 2> $D/bench_ref_n1.err
timeout 600 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $D/bench_short.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $D/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $D/ncu_launches.log 2>&1
python tools/ncu_launch_shares.py $D/launches.csv $D/launch_shares.txt > /dev/null 2>&1
tail -2 $D/tests.log $D/tests_attn_big.log; cat $D/attn_prev_order.jsonl $D/attn_lockstep.jsonl | cut -c1-200; head -20 $D/launch_shares.txt
