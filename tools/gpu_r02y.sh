# round 2, call y: DRAM traffic of the GEMM over the bench's own launch mix (ncu metrics pass over
# the first 800 gemm2 launches of `bench.py`), after the same command exited 0 without ncu
set -x
D=gpurun_out/r02y
mkdir -p $D
timeout 900 python bench.py --steps 2 --warmup 3 > $D/bench_plain.json 2> $D/bench_plain.err && \
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32.sum \
  --clock-control none -k regex:gemm2_kernel -c 800 --csv --page raw --log-file $D/ncu_gemm_bench_mix.csv \
  python bench.py --steps 2 --warmup 3 > $D/ncu_bench.log 2>&1
tail -2 $D/bench_plain.json; tail -3 $D/ncu_bench.log; wc -l $D/ncu_gemm_bench_mix.csv
python tools/ncu_traffic.py $D/ncu_gemm_bench_mix.csv $D/ncu_traffic_bench.json "ncu --metrics (dram read/write, tensor ops, duration) --clock-control none over the first 800 gemm2 launches of python bench.py --steps 2 --warmup 3 (N=1, the bench's own launch mix)" | head -20
gzip -k $D/ncu_gemm_bench_mix.csv
