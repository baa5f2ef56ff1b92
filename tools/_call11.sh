timeout 1500 python -m pytest tests -m gpu -q -x -rs > gpurun_out/r02_gpu_tests_1gpu_final.log 2>&1
echo "EXIT $?" >> gpurun_out/r02_gpu_tests_1gpu_final.log
SESGD_LIB=checked timeout 1500 python -m pytest tests/test_gpu_multigpu.py tests/test_gpu_stats.py tests/test_gpu_resident.py -m gpu -q -x > gpurun_out/r02_gpu_tests_checked.log 2>&1
echo "EXIT $?" >> gpurun_out/r02_gpu_tests_checked.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke_final.log 2>&1
timeout 400 python bench.py > gpurun_out/r02_bench_g1_final.json 2> gpurun_out/r02_bench_g1_final.err
echo done
