# call 20 (1 GPU): final-build evidence -- full GPU suite (loopback), checked build, smoke, bench, ncu
export PYTEST_ADDOPTS="-p no:cacheprovider"
timeout 1800 python -m pytest tests -m gpu -q -rs --timeout 600 > gpurun_out/r02_c20_gpu_tests_1gpu.log 2>&1
echo "EXIT $?" >> gpurun_out/r02_c20_gpu_tests_1gpu.log
SESGD_LIB=checked timeout 1200 python -m pytest tests/test_gpu_multigpu.py tests/test_gpu_stats.py tests/test_gpu_resident.py -m gpu -q --timeout 600 -k "device_iteration or k4w or pair_harness or resnet50" > gpurun_out/r02_c20_gpu_tests_checked.log 2>&1
echo "EXIT $?" >> gpurun_out/r02_c20_gpu_tests_checked.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_c20_smoke.log 2>&1
echo "EXIT $?" >> gpurun_out/r02_c20_smoke.log
timeout 600 python bench.py > gpurun_out/r02_c20_bench_g1.json 2> gpurun_out/r02_c20_bench_g1.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_c20_launches_g1.csv python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline --second-workload 0 > gpurun_out/r02_c20_ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k4w_multi_pair -s 3 -c 1 -o gpurun_out/r02_c20_k4wm_pair python tools/k4w_pair_profile.py 4 8 > gpurun_out/r02_c20_ncu_k4wm.log 2>&1
echo done
