B="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29500 --nproc-per-node 2"
export PYTEST_ADDOPTS="-p no:cacheprovider"
timeout 900 python -m pytest tests/test_gpu_multigpu.py tests/test_gpu_stats.py -m gpu -q -x --timeout 300 -k "k4w_multi or pair_harness or (device_iteration and 8)" > gpurun_out/r02_c19_tests.log 2>&1
echo "EXIT $?" >> gpurun_out/r02_c19_tests.log
timeout 200 $B bench.py --gpus 2 --steps 100 --warmup 10 --e2e-steps 0 --second-workload 0 --no-cpu-baseline > gpurun_out/r02_c19_bench_g2.json 2>/dev/null
timeout 150 $B tools/k3_phase_profile.py --workers 8 --path 4 --protocol 2 --out gpurun_out/r02_c19_k4wm_phases.json > /dev/null 2>&1
timeout 200 $B bench.py --gpus 2 --workers 4 --protocol 2 --steps 100 --warmup 10 --e2e-steps 0 --second-workload 0 --no-cpu-baseline > gpurun_out/r02_c19_bench_g2_n4_p2.json 2>/dev/null
timeout 300 python tools/k4w_pair_profile.py 20 8 > gpurun_out/r02_c19_pair.json 2>/dev/null
echo done
