# round 2, call p: the full single-GPU test tier + smoke on the final tree; ncu of the step kernels
set -x
D=gpurun_out/r02p
mkdir -p $D
python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > $D/gpu_tests.log 2>&1
python tools/ncu_step_kernels.py > $D/plain.log 2>&1 && \
ncu --set full --metrics sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32.sum,sm__inst_executed_pipe_tc.sum --clock-control none --import-source on \
    -k regex:"gemm2_kernel|attn_fwd_kernel|attn_bwd_kernel|fetch_tma_kernel|push_bulk_kernel|adam_kernel|slot_reduce" \
    -o /tmp/ncu_step_kernels python tools/ncu_step_kernels.py > $D/ncu.log 2>&1
cp gpurun_out/ncu_gemm_launches.json $D/ 2>/dev/null
ncu -i /tmp/ncu_step_kernels.ncu-rep --page raw --csv > $D/ncu_step_raw.csv 2>&1
ncu -i /tmp/ncu_step_kernels.ncu-rep --page details --csv -k regex:attn_bwd_kernel -c 1 > $D/ncu_attn_bwd_details.csv 2>&1
ls -la /tmp/ncu_step_kernels.ncu-rep
SZ=$(stat -c %s /tmp/ncu_step_kernels.ncu-rep 2>/dev/null || echo 0)
if [ "$SZ" -lt 25000000 ]; then cp /tmp/ncu_step_kernels.ncu-rep $D/; fi
for f in $D/*.csv; do [ $(stat -c %s $f) -gt 20000000 ] && gzip $f; done
du -sh gpurun_out
tail -3 $D/smoke.log $D/gpu_tests.log
