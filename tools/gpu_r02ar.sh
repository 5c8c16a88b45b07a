# round 2, call ar: ncu --set full of the step kernels on the FINAL tree (attention backward with the round-2
# schedule), after the same command exited 0 without ncu
set -x
D=gpurun_out/r02ar
mkdir -p $D
python tools/ncu_step_kernels.py > $D/plain.log 2>&1 && \
ncu --set full --metrics sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32.sum,sm__inst_executed_pipe_tc.sum --clock-control none --import-source on \
    -k regex:"gemm2_kernel|attn_fwd_kernel|attn_bwd_kernel|fetch_tma_kernel|push_bulk_kernel|adam_kernel|slot_reduce" \
    -o /tmp/ncu_step_kernels python tools/ncu_step_kernels.py > $D/ncu.log 2>&1
cp gpurun_out/ncu_gemm_launches.json $D/ 2>/dev/null
ncu -i /tmp/ncu_step_kernels.ncu-rep --page raw --csv > $D/ncu_step_raw.csv 2>&1
ncu -i /tmp/ncu_step_kernels.ncu-rep --page details --csv -k regex:attn_bwd_kernel -c 1 > $D/ncu_attn_bwd_details.csv 2>&1
SZ=$(stat -c %s /tmp/ncu_step_kernels.ncu-rep 2>/dev/null || echo 0)
if [ "$SZ" -lt 25000000 ]; then cp /tmp/ncu_step_kernels.ncu-rep $D/; fi
for f in $D/*.csv; do [ $(stat -c %s $f) -gt 20000000 ] && gzip $f; done
tail -2 $D/ncu.log; ls -la $D
