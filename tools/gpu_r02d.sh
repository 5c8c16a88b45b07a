# round 2, call d: local-group deadlock debug, attention v2 vs v3 A/B (same box), fused SwiGLU test, L2 budget sweep
set -x
mkdir -p gpurun_out/r02d
for c in "fixed 2" "slot 2" "red 4"; do timeout 120 python tools/lg_debug.py $c > "gpurun_out/r02d/lg_${c// /_}.log" 2>&1; done
(cd _ab/v2 && timeout 300 python attn_bwd_ab.py) > gpurun_out/r02d/attn_v2.jsonl 2>&1
ODC_ATTN_DQ=tma timeout 300 python tools/attn_bwd_ab.py > gpurun_out/r02d/attn_v3_tma.jsonl 2>&1
timeout 600 python -m pytest tests/test_gemm_gpu.py tests/test_worker_gpu.py -q --timeout 300 -p no:cacheprovider > gpurun_out/r02d/tests.log 2>&1
for mb in 20 80 160; do ODC_GEMM_L2_MB=$mb timeout 300 python tools/gemm_raster_ab.py > gpurun_out/r02d/gemm_l2_$mb.jsonl 2>&1; done
tail -3 gpurun_out/r02d/tests.log
