# round 2, call af: SM-clock timeline of the shipped attention backward (trace build), 32K and 64K
set -x
D=gpurun_out/r02af
mkdir -p $D
ODC_LIB_PATH=paper_2601_19362_b200/lib/variants/trace/libodc.so timeout -s KILL 120 python tools/attn_bwd_trace.py > $D/trace_32k.txt 2>&1
cat $D/trace_32k.txt
timeout -s KILL 300 python -m pytest tests/test_attention_gpu.py -q -x --timeout 240 -p no:cacheprovider > $D/tests.log 2>&1
tail -n 1 $D/tests.log
