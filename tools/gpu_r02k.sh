# round 2, call k: fused SwiGLU-bwd + fetch pipeline verification, config0 (both arms), N=1 bench,
# MMA probe, ncu of the step kernels (raw CSV kept; the .ncu-rep only if small enough to bring back)
set -x
D=gpurun_out/r02k
mkdir -p $D
./tools/tmem_probe > $D/tmem_probe.txt 2>&1
timeout 1200 python -m pytest tests/test_gemm_gpu.py tests/test_attention_gpu.py tests/test_worker_gpu.py tests/test_engine_gpu.py tests/test_engine_local_group_gpu.py tests/test_fabric_gpu.py tests/test_config0_gpu.py tests/test_bench_config_gpu.py -q --timeout 900 -p no:cacheprovider > $D/tests.log 2>&1
timeout 600 python bench.py --workload config0 --steps 20 --warmup 5 > $D/config0.json 2> $D/config0.err
timeout 600 python bench.py --workload config0 --impl reference --steps 5 --warmup 1 > $D/config0_ref.json 2> $D/config0_ref.err
timeout 900 python bench.py > $D/bench_n1.json 2> $D/bench_n1.err
python tools/ncu_step_kernels.py > $D/plain.log 2>&1 && \
ncu --set full --metrics sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32.sum,sm__inst_executed_pipe_tc.sum --clock-control none --import-source on \
    -k regex:"gemm2_kernel|attn_fwd_kernel|attn_bwd_kernel|fetch_tma_kernel|push_bulk_kernel|adam_kernel" \
    -o /tmp/ncu_step_kernels python tools/ncu_step_kernels.py > $D/ncu.log 2>&1
cp gpurun_out/ncu_gemm_launches.json $D/ 2>/dev/null
ncu -i /tmp/ncu_step_kernels.ncu-rep --page raw --csv > $D/ncu_step_raw.csv 2>&1
ncu -i /tmp/ncu_step_kernels.ncu-rep --page source --csv -k regex:attn_bwd_kernel -c 1 > $D/ncu_attn_bwd_source.csv 2>&1
ls -la /tmp/ncu_step_kernels.ncu-rep
SZ=$(stat -c %s /tmp/ncu_step_kernels.ncu-rep 2>/dev/null || echo 0)
if [ "$SZ" -lt 30000000 ]; then cp /tmp/ncu_step_kernels.ncu-rep $D/; fi
for f in $D/ncu_attn_bwd_source.csv $D/ncu_step_raw.csv; do [ $(stat -c %s $f) -gt 20000000 ] && gzip $f; done
du -sh gpurun_out
tail -3 $D/tests.log; tail -3 $D/ncu.log
