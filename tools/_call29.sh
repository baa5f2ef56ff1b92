# call 29 (1 GPU): the full GPU suite at the final code, as the driver runs it
export PYTEST_ADDOPTS="-p no:cacheprovider"
timeout 2400 python -m pytest tests -x -q -m gpu -rs > gpurun_out/r02_c29_gpu_tests_final.log 2>&1
echo "EXIT $?" >> gpurun_out/r02_c29_gpu_tests_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_c29_smoke.log 2>&1
echo "EXIT $?" >> gpurun_out/r02_c29_smoke.log
echo done
