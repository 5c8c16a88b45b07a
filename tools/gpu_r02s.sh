# round 2, call s: timeline of the transposed-score attention backward (trace build)
set -x
D=gpurun_out/r02s
mkdir -p $D
ODC_ATTN_BWD=t ODC_LIB_PATH=paper_2601_19362_b200/lib/variants/trace/libodc.so timeout -s KILL 300 python tools/attn_bwd_trace.py > $D/trace_32k.txt 2>&1
cat $D/trace_32k.txt
