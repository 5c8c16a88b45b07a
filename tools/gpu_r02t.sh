# round 2, call t: transposed-score attention backward with deferred staging drains: parity, trace, A/B
set -x
D=gpurun_out/r02t
mkdir -p $D
timeout -s KILL 300 python -m pytest tests/test_attention_gpu.py -q -x -k bwd --timeout 240 -p no:cacheprovider > $D/tests_t.log 2>&1
tail -2 $D/tests_t.log
ODC_ATTN_BWD=t ODC_LIB_PATH=paper_2601_19362_b200/lib/variants/trace/libodc.so timeout -s KILL 120 python tools/attn_bwd_trace.py > $D/trace_32k.txt 2>&1
cat $D/trace_32k.txt
if grep -q " passed" $D/tests_t.log && ! grep -q "failed" $D/tests_t.log; then
  timeout -s KILL 600 python -m pytest tests/test_bench_config_gpu.py -q -x -k "attention_long or one_32k" --timeout 500 -p no:cacheprovider > $D/tests_t_long.log 2>&1
  tail -2 $D/tests_t_long.log
  for v in v2 t v2 t; do ODC_ATTN_BWD=$v timeout -s KILL 300 python tools/attn_bwd_ab.py >> $D/attn_ab.jsonl 2>&1; done
  grep '^{' $D/attn_ab.jsonl | cut -c1-220
fi
