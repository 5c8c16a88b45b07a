# round 2, call h: ncu evidence of the final tree (step kernels at N=1) + a step launch list
set -x
mkdir -p gpurun_out/r02h
python tools/ncu_step_kernels.py > gpurun_out/r02h/plain.log 2>&1 && \
ncu --set full --metrics sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32.sum,sm__inst_executed_pipe_tc.sum --clock-control none --import-source on \
    -k regex:"gemm2_kernel|attn_fwd_kernel|attn_bwd_kernel|fetch_tma_kernel|push_bulk_kernel|adam_kernel" \
    -o gpurun_out/r02h/ncu_step_kernels python tools/ncu_step_kernels.py > gpurun_out/r02h/ncu.log 2>&1
cp gpurun_out/ncu_gemm_launches.json gpurun_out/r02h/ 2>/dev/null
tail -3 gpurun_out/r02h/ncu.log
