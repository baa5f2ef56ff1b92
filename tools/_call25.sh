# call 25 (2 GPUs): final build -- full loopback suite, 2-GPU NVLink K4W-M / device-iteration / DDP subset,
# bounds-checked subset, smoke, bench N=1 and N=2, K4W-M phases
export PYTEST_ADDOPTS="-p no:cacheprovider"
timeout 1800 python -m pytest tests -m gpu -q -rs --timeout 600 -k "not nvlink" > gpurun_out/r02_c25_gpu_tests_loopback.log 2>&1
echo "EXIT $?" >> gpurun_out/r02_c25_gpu_tests_loopback.log
timeout 1200 python -m pytest tests/test_gpu_multigpu.py tests/test_gpu_ddp.py -m gpu -q -rs --timeout 600 -k "nvlink and (k4w or device_iteration or two_gpus_value_protocol or resnet50)" > gpurun_out/r02_c25_gpu_tests_nvlink2.log 2>&1
echo "EXIT $?" >> gpurun_out/r02_c25_gpu_tests_nvlink2.log
SESGD_LIB=checked timeout 900 python -m pytest tests/test_gpu_multigpu.py tests/test_gpu_stats.py tests/test_gpu_resident.py -m gpu -q --timeout 600 -k "(device_iteration or k4w_multi or pair_harness) and not nvlink" > gpurun_out/r02_c25_gpu_tests_checked.log 2>&1
echo "EXIT $?" >> gpurun_out/r02_c25_gpu_tests_checked.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_c25_smoke.log 2>&1
echo "EXIT $?" >> gpurun_out/r02_c25_smoke.log
timeout 600 python bench.py > gpurun_out/r02_c25_bench_g1.json 2> gpurun_out/r02_c25_bench_g1.err
B="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29500 --nproc-per-node 2"
timeout 600 $B bench.py --gpus 2 --steps 100 --warmup 10 > gpurun_out/r02_c25_bench_g2.json 2> gpurun_out/r02_c25_bench_g2.err
timeout 150 $B tools/k3_phase_profile.py --workers 8 --path 4 --protocol 2 --out gpurun_out/r02_c25_k4wm_phases.json > /dev/null 2>&1
echo done
