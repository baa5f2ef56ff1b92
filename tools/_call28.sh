# call 28 (4 GPUs): ResNet-50 training bench, SESGD eager vs one captured training-step graph vs torch DDP
T4="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29500 --nproc-per-node 4"
T2="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29501 --nproc-per-node 2"
timeout 900 $T4 tools/train_bench.py --arms compute,sesgd,sesgd_graph,ddp --batch 32 --steps 30 --warmup 8 --out gpurun_out/r02_c28_train_g4_b32.json > gpurun_out/r02_c28_train_g4_b32.log 2>&1
timeout 900 $T4 tools/train_bench.py --arms compute,sesgd,sesgd_graph,ddp --batch 64 --steps 30 --warmup 8 --out gpurun_out/r02_c28_train_g4_b64.json > gpurun_out/r02_c28_train_g4_b64.log 2>&1
timeout 900 $T2 tools/train_bench.py --arms compute,sesgd,sesgd_graph,ddp --batch 32 --steps 30 --warmup 8 --gsize 2 --out gpurun_out/r02_c28_train_g2_b32.json > gpurun_out/r02_c28_train_g2_b32.log 2>&1
echo done
