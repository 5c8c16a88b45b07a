# round 2, call w: paired-CTA (DSMEM dQ exchange) transposed attention backward: parity, trace, A/B
set -x
D=gpurun_out/r02w
mkdir -p $D
ODC_ATTN_BWD=t timeout -s KILL 300 python -m pytest tests/test_attention_gpu.py -q -x -k "bwd" --timeout 240 -p no:cacheprovider > $D/tests_t.log 2>&1
tail -n 2 $D/tests_t.log
ODC_ATTN_BWD=t ODC_LIB_PATH=paper_2601_19362_b200/lib/variants/trace/libodc.so timeout -s KILL 120 python tools/attn_bwd_trace.py > $D/trace_32k.txt 2>&1
cat $D/trace_32k.txt
for v in v2 t nopoly v2 t nopoly; do
  if [ $v = nopoly ]; then L=paper_2601_19362_b200/lib/variants/nopoly/libodc.so; V=t; else L=paper_2601_19362_b200/lib/libodc.so; V=$v; fi
  ODC_LIB_PATH=$L ODC_ATTN_BWD=$V timeout -s KILL 300 python tools/attn_bwd_ab.py | sed "s/\"variant\": \"t\"/\"variant\": \"$v\"/" >> $D/attn_ab.jsonl 2>&1
done
grep '^{' $D/attn_ab.jsonl | cut -c1-200
