# round 2, call al (4 GPUs): device-restoring C-ABI calls: the engine/fabric/world-8 tests on 4 GPUs
set -x
D=gpurun_out/r02al
mkdir -p $D
timeout 1500 python -m pytest tests/test_engine_gpu.py tests/test_engine_multigpu.py tests/test_worker_multigpu.py tests/test_engine_local_group_gpu.py tests/test_fabric_gpu.py tests/test_world8_step_gpu.py tests/test_config0_gpu.py tests/test_refsuite.py -q --timeout 900 -p no:cacheprovider > $D/tests.log 2>&1
tail -n 3 $D/tests.log
