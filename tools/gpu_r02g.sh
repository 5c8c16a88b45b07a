# round 2, call g: protocol tests with per-stream gate kernels; compute-sanitizer memcheck; N=1 bench
set -x
mkdir -p gpurun_out/r02g
timeout 1200 python -m pytest tests/test_engine_local_group_gpu.py tests/test_config0_gpu.py tests/test_engine_gpu.py tests/test_fabric_gpu.py tests/test_worker_gpu.py tests/test_gemm_gpu.py -q --timeout 600 -p no:cacheprovider > gpurun_out/r02g/tests.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02g/bench_n1.json 2> gpurun_out/r02g/bench_n1.err
timeout 900 compute-sanitizer --tool memcheck --print-limit 50 python tools/sanitize_protocol.py > gpurun_out/r02g/sanitizer_memcheck.log 2>&1
tail -3 gpurun_out/r02g/tests.log; tail -5 gpurun_out/r02g/sanitizer_memcheck.log
