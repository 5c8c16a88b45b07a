# round 2, call r: transposed-score attention backward (attn_bwd_t_kernel): parity, then A/B timing vs v2
set -x
D=gpurun_out/r02r
mkdir -p $D
timeout -s KILL 300 python -m pytest tests/test_attention_gpu.py -q -x -k bwd --timeout 240 -p no:cacheprovider > $D/tests_t.log 2>&1
tail -3 $D/tests_t.log
if grep -q " passed" $D/tests_t.log && ! grep -q "failed" $D/tests_t.log; then
  timeout -s KILL 600 python -m pytest tests/test_bench_config_gpu.py -q -x -k "attention_long or one_32k" --timeout 500 -p no:cacheprovider > $D/tests_t_long.log 2>&1
  tail -3 $D/tests_t_long.log
  for v in v2 t v2 t; do ODC_ATTN_BWD=$v timeout -s KILL 300 python tools/attn_bwd_ab.py >> $D/attn_ab.jsonl 2>&1; done
  grep '^{' $D/attn_ab.jsonl | cut -c1-220
fi
