# round 2, call ap: final-tree verification (parameterised attention backward) on one B200: smoke, the full -m gpu tier, the default bench
# (20 steps, 5 warm-up) and the reference arm, as the driver runs them
set -x
D=gpurun_out/r02ap
mkdir -p $D
python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > $D/gpu_tests.log 2>&1
timeout 1800 python bench.py > $D/bench_n1.json 2> $D/bench_n1.err
timeout 1200 python bench.py --impl reference > $D/bench_ref_n1.json 2> $D/bench_ref_n1.err
tail -n 2 $D/smoke.log $D/gpu_tests.log; cat $D/bench_n1.json $D/bench_ref_n1.json | cut -c1-400
