# round 2, call as: attention backward: P_n starts on S_n alone (s_full), before dP_n is done; vs HEAD (prev)
set -x
D=gpurun_out/r02as
mkdir -p $D
timeout -s KILL 300 python -m pytest tests/test_attention_gpu.py -q -x --timeout 240 -p no:cacheprovider > $D/tests.log 2>&1
tail -n 1 $D/tests.log
for v in earlyp prev earlyp prev earlyp prev; do
  if [ $v = prev ]; then L=paper_2601_19362_b200/lib/variants/prev/libodc.so; else L=paper_2601_19362_b200/lib/libodc.so; fi
  ODC_LIB_PATH=$L ODC_ATTN_BWD=$v timeout -s KILL 300 python tools/attn_bwd_ab.py >> $D/attn_ab.jsonl 2>&1
done
grep -o '"T": [0-9]*, "H": [0-9]*.*"variant": "[a-z0-9]*", "bwd_ms": [0-9.]*, "bwd_tflops": [0-9.]*' $D/attn_ab.jsonl
ODC_LIB_PATH=paper_2601_19362_b200/lib/variants/trace/libodc.so timeout -s KILL 120 python tools/attn_bwd_trace.py > $D/trace_32k.txt 2>&1; head -1 $D/trace_32k.txt | cut -c1-80
