# round 2, call l: final-tree N=1 bench + the ncu launch list of the same bench command
set -x
D=gpurun_out/r02l
mkdir -p $D
timeout 900 python bench.py > $D/bench_n1.json 2> $D/bench_n1.err
timeout 900 python bench.py --impl reference > $D/bench_ref_n1.json 2> $D/bench_ref_n1.err
timeout 600 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $D/bench_short.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $D/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $D/ncu_launches.log 2>&1
python tools/ncu_launch_shares.py $D/launches.csv $D/launch_shares.txt > /dev/null 2>&1
cat $D/launch_shares.txt | head -30
