# round 2, call f: local-group protocol after kernel preloading, config0, fused SwiGLU worker tests, raster A/B (interleaved)
set -x
mkdir -p gpurun_out/r02f
for c in "fixed 2" "slot 2"; do timeout 120 python tools/lg_debug.py $c > "gpurun_out/r02f/lg_${c// /_}.log" 2>&1; done
timeout 1200 python -m pytest tests/test_engine_local_group_gpu.py tests/test_config0_gpu.py tests/test_engine_gpu.py tests/test_worker_gpu.py tests/test_refsuite.py -q --timeout 600 -p no:cacheprovider > gpurun_out/r02f/tests.log 2>&1
timeout 900 python tools/gemm_raster_ab.py 5 5 > gpurun_out/r02f/raster_ab.jsonl 2>&1
tail -3 gpurun_out/r02f/tests.log
