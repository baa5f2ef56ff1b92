# call 21 (4 GPUs): NVLink-transport suite, multi-GPU bench lines (same-box protocol A/B), per-layer sweep
export PYTEST_ADDOPTS="-p no:cacheprovider"
timeout 2400 python -m pytest tests/test_gpu_multigpu.py tests/test_gpu_ddp.py -m gpu -q -rs --timeout 900 -k "nvlink or ddp" > gpurun_out/r02_c21_gpu_tests_4gpu.log 2>&1
echo "EXIT $?" >> gpurun_out/r02_c21_gpu_tests_4gpu.log
T4="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29500 --nproc-per-node 4"
T2="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29501 --nproc-per-node 2"
timeout 600 $T4 bench.py --gpus 4 --steps 100 --warmup 10 > gpurun_out/r02_c21_bench_g4.json 2> gpurun_out/r02_c21_bench_g4.err
timeout 600 $T2 bench.py --gpus 2 --steps 100 --warmup 10 > gpurun_out/r02_c21_bench_g2.json 2> gpurun_out/r02_c21_bench_g2.err
for rep in 1 2; do
for p in 1 2; do
timeout 200 $T2 bench.py --gpus 2 --steps 100 --warmup 10 --e2e-steps 0 --second-workload 0 --no-cpu-baseline --protocol $p > gpurun_out/r02_c21_ab_g2_n8_p${p}_r$rep.json 2>/dev/null
timeout 200 $T2 bench.py --gpus 2 --workers 4 --steps 100 --warmup 10 --e2e-steps 0 --second-workload 0 --no-cpu-baseline --protocol $p > gpurun_out/r02_c21_ab_g2_n4_p${p}_r$rep.json 2>/dev/null
timeout 200 $T4 bench.py --gpus 4 --steps 100 --warmup 10 --e2e-steps 0 --second-workload 0 --no-cpu-baseline --protocol $p > gpurun_out/r02_c21_ab_g4_n8_p${p}_r$rep.json 2>/dev/null
done
done
timeout 200 $T2 bench.py --gpus 2 --steps 100 --warmup 10 --e2e-steps 0 --second-workload 0 --no-cpu-baseline --protocol 2 --experiment 2 > gpurun_out/r02_c21_exp2_g2_n8_p2.json 2>/dev/null
timeout 200 $T4 bench.py --gpus 4 --workers 4 --steps 200 --warmup 10 --e2e-steps 0 --second-workload 0 --no-cpu-baseline > gpurun_out/r02_c21_bench_g4_n4_k4w.json 2>/dev/null
timeout 1200 $T4 tools/per_layer_sweep.py --hops-us 0,100,5000 --out gpurun_out/r02_c21_per_layer_sweep_4gpu.json > gpurun_out/r02_c21_per_layer.log 2>&1
echo done
