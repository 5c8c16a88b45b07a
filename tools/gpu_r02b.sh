# round 2, call b: new protocol tests + probes + GEMM raster A/B
set -x
mkdir -p gpurun_out/r02b
./tools/tmem_probe > gpurun_out/r02b/tmem_probe.txt 2>&1
timeout 1500 python -m pytest tests/test_engine_local_group_gpu.py tests/test_config0_gpu.py tests/test_worker_gpu.py tests/test_engine_gpu.py tests/test_gemm_gpu.py tests/test_bench_config_gpu.py -q --timeout 900 -p no:cacheprovider > gpurun_out/r02b/tests.log 2>&1
ODC_GEMM_GROUP=8 timeout 300 python tools/gemm_raster_ab.py > gpurun_out/r02b/gemm_group8.jsonl 2>&1
timeout 300 python tools/gemm_raster_ab.py > gpurun_out/r02b/gemm_auto.jsonl 2>&1
ODC_GEMM_GROUP=8 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:gemm --csv --log-file gpurun_out/r02b/ncu_gemm_group8.csv python tools/gemm_raster_ab.py 1 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:gemm --csv --log-file gpurun_out/r02b/ncu_gemm_auto.csv python tools/gemm_raster_ab.py 1 > /dev/null 2>&1
tail -5 gpurun_out/r02b/tests.log
