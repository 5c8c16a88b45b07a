# round 2, call o: attention-backward variant A/B (same box) + attention parity per variant
set -x
D=gpurun_out/r02o
mkdir -p $D
for v in 0 1 2 3 0; do ODC_ATTN_BWD_VAR=$v timeout 300 python tools/attn_bwd_ab.py > $D/attn_var$v.jsonl 2>&1; done
for v in 1 2 3; do ODC_ATTN_BWD_VAR=$v timeout 600 python -m pytest tests/test_attention_gpu.py -q -k bwd --timeout 300 -p no:cacheprovider > $D/tests_var$v.log 2>&1; done
for v in 0 1 2 3; do echo var $v; grep '^{' $D/attn_var$v.jsonl | cut -c1-160; done; tail -1 $D/tests_var*.log
for k in 1 2 3 4 5; do timeout 600 python -m pytest tests/test_engine_local_group_gpu.py -q --timeout 300 -p no:cacheprovider > $D/lg_rep$k.log 2>&1; done
tail -1 $D/lg_rep*.log
