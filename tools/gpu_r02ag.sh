# round 2, call ag: attention backward: S read out alone before P (dP later), and the exp2 of P on
# MUFU f32 (exp0, default build) / 1 pair in 4 on the FMA pipe (exp1) / MUFU f16x2 (exp2), vs HEAD (prev)
set -x
D=gpurun_out/r02ag
mkdir -p $D
for v in exp0 exp2; do
  if [ $v = exp0 ]; then L=paper_2601_19362_b200/lib/libodc.so; else L=paper_2601_19362_b200/lib/variants/$v/libodc.so; fi
  ODC_LIB_PATH=$L timeout -s KILL 300 python -m pytest tests/test_attention_gpu.py -q -x --timeout 240 -p no:cacheprovider > $D/tests_$v.log 2>&1
  tail -n 1 $D/tests_$v.log
done
for v in exp0 prev exp1 exp2 exp0 prev exp1 exp2; do
  if [ $v = exp0 ]; then L=paper_2601_19362_b200/lib/libodc.so; else L=paper_2601_19362_b200/lib/variants/$v/libodc.so; fi
  ODC_LIB_PATH=$L ODC_ATTN_BWD=$v timeout -s KILL 300 python tools/attn_bwd_ab.py >> $D/attn_ab.jsonl 2>&1
done
grep -o '"T": [0-9]*, "H": [0-9]*.*"variant": "[a-z0-9]*", "bwd_ms": [0-9.]*, "bwd_tflops": [0-9.]*' $D/attn_ab.jsonl
