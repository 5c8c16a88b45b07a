# round 2, call at (4 GPUs): fetch TMA ring A/B: 32 KB x 5 (shipped), 64 KB x 3, 16 KB x 9, 32 KB x 7
set -x
D=gpurun_out/r02at
mkdir -p $D
P=29640
for v in base f64x3 f16x9 f32x7 base; do
  if [ $v = base ]; then L=paper_2601_19362_b200/lib/libodc.so; else L=paper_2601_19362_b200/lib/variants/$v/libodc.so; fi
  P=$((P+1))
  ODC_LIB_PATH=$L timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $P bench_p2p.py --sizes 4M,16M,32M,64M --out $D/p2p_$v.md > $D/p2p_$v.jsonl 2> $D/p2p_$v.err
  echo $v; grep '"odc_fetch"' $D/p2p_$v.jsonl | cut -c1-120
done
