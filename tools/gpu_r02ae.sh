# round 2, call ae: attention backward with dQ issued before dK (its read-out overlaps dK; each
# elementwise warpgroup stages and reduces its own dQ half) vs the previous build (lib/variants/prev)
set -x
D=gpurun_out/r02ae
mkdir -p $D
timeout -s KILL 300 python -m pytest tests/test_attention_gpu.py -q -x --timeout 240 -p no:cacheprovider > $D/tests.log 2>&1
tail -n 2 $D/tests.log
for v in dqfirst prev dqfirst prev dqfirst prev; do
  if [ $v = prev ]; then L=paper_2601_19362_b200/lib/variants/prev/libodc.so; else L=paper_2601_19362_b200/lib/libodc.so; fi
  ODC_LIB_PATH=$L ODC_ATTN_BWD=$v timeout -s KILL 300 python tools/attn_bwd_ab.py >> $D/attn_ab.jsonl 2>&1
done
grep -o '"T": [0-9]*, "H": [0-9]*.*"variant": "[a-z0-9]*", "bwd_ms": [0-9.]*, "bwd_tflops": [0-9.]*' $D/attn_ab.jsonl
