# call 23 (2 GPUs): K4W-M S with paired spanning items; parity subset; same-box A/B vs K4
export PYTEST_ADDOPTS="-p no:cacheprovider"
B="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29500 --nproc-per-node 2"
for rep in 1 2; do
timeout 200 $B bench.py --gpus 2 --steps 100 --warmup 10 --e2e-steps 0 --second-workload 0 --no-cpu-baseline --protocol 2 > gpurun_out/r02_c23_g2_n8_p2_r$rep.json 2>/dev/null
timeout 200 $B bench.py --gpus 2 --steps 100 --warmup 10 --e2e-steps 0 --second-workload 0 --no-cpu-baseline --protocol 1 > gpurun_out/r02_c23_g2_n8_p1_r$rep.json 2>/dev/null
timeout 200 $B bench.py --gpus 2 --workers 4 --steps 100 --warmup 10 --e2e-steps 0 --second-workload 0 --no-cpu-baseline --protocol 2 > gpurun_out/r02_c23_g2_n4_p2_r$rep.json 2>/dev/null
timeout 200 $B bench.py --gpus 2 --workers 4 --steps 100 --warmup 10 --e2e-steps 0 --second-workload 0 --no-cpu-baseline --protocol 1 > gpurun_out/r02_c23_g2_n4_p1_r$rep.json 2>/dev/null
done
timeout 150 $B tools/k3_phase_profile.py --workers 8 --path 4 --protocol 2 --out gpurun_out/r02_c23_k4wm_phases.json > /dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_multigpu.py tests/test_gpu_stats.py tests/test_gpu_ddp.py -m gpu -q -rs --timeout 600 -k "(k4w_multi or pair_harness or loopback_replicas or (device_iteration and 8)) and not nvlink" > gpurun_out/r02_c23_tests.log 2>&1
echo "EXIT $?" >> gpurun_out/r02_c23_tests.log
echo done
