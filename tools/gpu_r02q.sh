# round 2, call q: the world-8 single-process SFT step test (noise-floor check)
set -x
D=gpurun_out/r02q
mkdir -p $D
timeout 1200 python -m pytest tests/test_world8_step_gpu.py -q -s --timeout 900 -p no:cacheprovider > $D/world8.log 2>&1
tail -40 $D/world8.log
