timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 tests/ddp_worker.py --gsize 2 --iters 6 --static 1 --graph 1 --out gpurun_out/r02_c31_log.npy > gpurun_out/r02_c31_worker.log 2>&1
echo "EXIT $?" >> gpurun_out/r02_c31_worker.log
echo done
