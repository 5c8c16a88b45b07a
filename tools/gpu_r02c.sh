# round 2, call c: attention bwd v3 (two-phase elementwise) A/B + parity; new SLOT; local-group protocol
set -x
mkdir -p gpurun_out/r02c
timeout 900 python -m pytest tests/test_attention_gpu.py tests/test_engine_local_group_gpu.py tests/test_engine_gpu.py tests/test_config0_gpu.py tests/test_fabric_gpu.py -q --timeout 600 -p no:cacheprovider > gpurun_out/r02c/tests.log 2>&1
timeout 900 python -m pytest tests/test_bench_config_gpu.py -q --timeout 900 -p no:cacheprovider -k attention > gpurun_out/r02c/tests_attn_big.log 2>&1
timeout 300 python tools/attn_bwd_ab.py > gpurun_out/r02c/attn_red.jsonl 2>&1
ODC_ATTN_DQ=tma timeout 300 python tools/attn_bwd_ab.py > gpurun_out/r02c/attn_tma.jsonl 2>&1
tail -3 gpurun_out/r02c/tests.log gpurun_out/r02c/tests_attn_big.log
