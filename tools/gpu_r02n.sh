# round 2, call n: the full single-GPU test tier on the final tree + smoke
set -x
D=gpurun_out/r02n
mkdir -p $D
python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > $D/gpu_tests.log 2>&1
tail -3 $D/smoke.log $D/gpu_tests.log
