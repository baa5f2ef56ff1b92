# call 22 (2 GPUs): hybrid K6 + K4W-M, loopback DDP, device-mode argument copy
export PYTEST_ADDOPTS="-p no:cacheprovider"
B="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29500 --nproc-per-node 2"
for rep in 1 2; do
timeout 200 $B bench.py --gpus 2 --steps 100 --warmup 10 --e2e-steps 0 --second-workload 0 --no-cpu-baseline > gpurun_out/r02_c22_g2_n8_hybrid_r$rep.json 2>/dev/null
timeout 200 $B bench.py --gpus 2 --steps 100 --warmup 10 --e2e-steps 0 --second-workload 0 --no-cpu-baseline --no-hybrid > gpurun_out/r02_c22_g2_n8_nohybrid_r$rep.json 2>/dev/null
timeout 200 $B bench.py --gpus 2 --steps 100 --warmup 10 --e2e-steps 0 --second-workload 0 --no-cpu-baseline --protocol 1 > gpurun_out/r02_c22_g2_n8_k4_r$rep.json 2>/dev/null
done
timeout 200 $B bench.py --gpus 2 --workers 4 --protocol 2 --steps 100 --warmup 10 --e2e-steps 0 --second-workload 0 --no-cpu-baseline > gpurun_out/r02_c22_g2_n4_hybrid.json 2>/dev/null
timeout 1500 python -m pytest tests/test_gpu_multigpu.py tests/test_gpu_stats.py tests/test_gpu_resident.py tests/test_gpu_ddp.py -m gpu -q -rs --timeout 600 -k "(k4w_multi or pair_harness or device_iteration or loopback_replicas) and not nvlink" > gpurun_out/r02_c22_tests.log 2>&1
echo "EXIT $?" >> gpurun_out/r02_c22_tests.log
timeout 600 python tools/per_layer_sweep.py --loopback 4 --hops-us 0 --iters 20 --out gpurun_out/r02_c22_per_layer_loop4.json > gpurun_out/r02_c22_per_layer.log 2>&1
echo done
