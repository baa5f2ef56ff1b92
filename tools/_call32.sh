# call 32 (2 GPUs): the NVLink-transport suite (2-GPU cases) at the final code
export PYTEST_ADDOPTS="-p no:cacheprovider"
timeout 2700 python -m pytest tests/test_gpu_multigpu.py tests/test_gpu_ddp.py -m gpu -q -rs --timeout 900 -k "nvlink or ddp" > gpurun_out/r02_c32_gpu_tests_nvlink_2gpu.log 2>&1
echo "EXIT $?" >> gpurun_out/r02_c32_gpu_tests_nvlink_2gpu.log
echo done
