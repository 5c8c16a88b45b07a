# round 2, call x (4 GPUs): P2P table with concurrent fetch + push (RED / SLOT) columns
set -x
D=gpurun_out/r02x
mkdir -p $D
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29611 bench_p2p.py --sizes 1M,4M,16M,32M,64M,256M --out $D/p2p_n4_conc.md > $D/p2p_n4_conc.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29612 bench_p2p.py --sizes 1M,4M,16M,32M,64M,256M --out $D/p2p_n2_conc.md > $D/p2p_n2_conc.log 2>&1
cat $D/p2p_n4_conc.md $D/p2p_n2_conc.md
tail -3 $D/p2p_n4_conc.log
