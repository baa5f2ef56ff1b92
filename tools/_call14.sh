# call 14 (2 GPUs): device-iteration parity (loopback), K4W / K4W-M after the spin / decode changes,
# pair timings, N = 2 bench (K4W-M auto vs K4 protocol 1), K4W n = m = 2 bench
export PYTEST_ADDOPTS="-p no:cacheprovider"
timeout 1200 python -m pytest tests/test_gpu_resident.py tests/test_gpu_multigpu.py tests/test_gpu_stats.py -m gpu -q -rs --timeout 300 -k "device_iteration or pair_harness or k4w" > gpurun_out/r02_c14_tests.log 2>&1
echo "EXIT $?" >> gpurun_out/r02_c14_tests.log
timeout 300 python tools/k4w_pair_profile.py 20 8 > gpurun_out/r02_c14_k4wm_pair_time.json 2> gpurun_out/r02_c14_pair.err
timeout 300 python tools/k4w_pair_profile.py 20 2 > gpurun_out/r02_c14_k4w_pair_time.json 2>> gpurun_out/r02_c14_pair.err
B="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29500 --nproc-per-node 2"
timeout 200 $B bench.py --gpus 2 --steps 100 --warmup 10 --e2e-steps 0 --second-workload 0 > gpurun_out/r02_c14_bench_g2.json 2> gpurun_out/r02_c14_bench_g2.err
timeout 200 $B bench.py --gpus 2 --steps 100 --warmup 10 --e2e-steps 0 --protocol 1 --second-workload 0 > gpurun_out/r02_c14_bench_g2_p1.json 2>/dev/null
timeout 150 $B tools/k3_phase_profile.py --workers 8 --path 4 --protocol 2 --out gpurun_out/r02_c14_k4wm_phases.json > /dev/null 2>&1
timeout 150 $B tools/k3_phase_profile.py --workers 2 --path 4 --protocol 2 --out gpurun_out/r02_c14_k4w_phases.json > /dev/null 2>&1
timeout 200 $B bench.py --gpus 2 --workers 2 --group-size 2 --steps 200 --warmup 10 --e2e-steps 0 --second-workload 0 > gpurun_out/r02_c14_bench_n2.json 2>/dev/null
echo done
