# round 2, call ad: attention backward with the elementwise work split into a P pass (stored, dV starts)
# and a dS pass, vs the single-loop split-store build (lib/variants/poly0 = previous source, no poly exp)
set -x
D=gpurun_out/r02ad
mkdir -p $D
timeout -s KILL 300 python -m pytest tests/test_attention_gpu.py -q -x --timeout 240 -p no:cacheprovider > $D/tests.log 2>&1
tail -n 2 $D/tests.log
for v in pfirst oneloop pfirst oneloop pfirst oneloop; do
  if [ $v = oneloop ]; then L=paper_2601_19362_b200/lib/variants/poly0/libodc.so; else L=paper_2601_19362_b200/lib/libodc.so; fi
  ODC_LIB_PATH=$L ODC_ATTN_BWD=$v timeout -s KILL 300 python tools/attn_bwd_ab.py >> $D/attn_ab.jsonl 2>&1
done
grep -o '"T": [0-9]*, "H": [0-9]*.*"variant": "[a-z0-9]*", "bwd_ms": [0-9.]*, "bwd_tflops": [0-9.]*' $D/attn_ab.jsonl
