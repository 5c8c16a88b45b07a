# round 2, call ao: attention backward with 4 elementwise warpgroups (32 columns per thread, 640 threads)
# vs the 2-warpgroup kernel: parity of both, then interleaved A/B
set -x
D=gpurun_out/r02ao
mkdir -p $D
timeout -s KILL 300 python -m pytest tests/test_attention_gpu.py -q -x --timeout 240 -p no:cacheprovider > $D/tests_ew2.log 2>&1
ODC_LIB_PATH=paper_2601_19362_b200/lib/variants/ew4/libodc.so timeout -s KILL 300 python -m pytest tests/test_attention_gpu.py -q -x --timeout 240 -p no:cacheprovider > $D/tests_ew4.log 2>&1
tail -n 1 $D/tests_ew2.log $D/tests_ew4.log
for v in ew4 ew2 ew4 ew2 ew4 ew2; do
  if [ $v = ew4 ]; then L=paper_2601_19362_b200/lib/variants/ew4/libodc.so; else L=paper_2601_19362_b200/lib/libodc.so; fi
  ODC_LIB_PATH=$L ODC_ATTN_BWD=$v timeout -s KILL 300 python tools/attn_bwd_ab.py >> $D/attn_ab.jsonl 2>&1
done
grep -o '"T": [0-9]*, "H": [0-9]*.*"variant": "[a-z0-9]*", "bwd_ms": [0-9.]*, "bwd_tflops": [0-9.]*' $D/attn_ab.jsonl
