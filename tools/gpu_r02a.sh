set -x
mkdir -p gpurun_out/r02a
(nproc; free -g; lscpu | head -20; nvidia-smi) > gpurun_out/r02a/host.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02a/smoke.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/r02a/gpu_tests.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02a/bench_n1.json 2> gpurun_out/r02a/bench_n1.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02a/ref_n1.json 2> gpurun_out/r02a/ref_n1.err
tail -3 gpurun_out/r02a/gpu_tests.log
