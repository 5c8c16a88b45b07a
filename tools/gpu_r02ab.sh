# round 2, call ab: attention backward with the P / dS stores split around the two halves of the dQ
# staging drain (dV starts on P): parity, then A/B against the single-store build
set -x
D=gpurun_out/r02ab
mkdir -p $D
timeout -s KILL 300 python -m pytest tests/test_attention_gpu.py -q -x --timeout 240 -p no:cacheprovider > $D/tests.log 2>&1
tail -n 2 $D/tests.log
for v in split nosplit split nosplit; do
  if [ $v = nosplit ]; then L=paper_2601_19362_b200/lib/variants/nosplit/libodc.so; else L=paper_2601_19362_b200/lib/libodc.so; fi
  ODC_LIB_PATH=$L ODC_ATTN_BWD=$v timeout -s KILL 300 python tools/attn_bwd_ab.py >> $D/attn_ab.jsonl 2>&1
done
grep -o '"T": [0-9]*, "H": [0-9]*.*"variant": "[a-z]*", "bwd_ms": [0-9.]*, "bwd_tflops": [0-9.]*' $D/attn_ab.jsonl
