# round 2, call z: device-busy share of one timed bench step: every kernel launched inside the first timed
# step (NVTX range odc_step) with its duration, vs the step's event time without ncu
set -x
D=gpurun_out/r02z
mkdir -p $D
ODC_BENCH_LOG=1 ODC_NVTX_STEP=1 timeout 900 python bench.py --steps 2 --warmup 3 > $D/bench_plain.json 2> $D/bench_plain.err && \
ODC_NVTX_STEP=1 timeout 1500 ncu --nvtx --nvtx-include "odc_step/" --metrics gpu__time_duration.sum --clock-control none \
  --csv --log-file $D/step_launches.csv python bench.py --steps 2 --warmup 3 > $D/ncu_bench.log 2>&1
grep "timed steps done" $D/bench_plain.err
python tools/ncu_launch_shares.py $D/step_launches.csv $D/step_shares.txt | head -30
