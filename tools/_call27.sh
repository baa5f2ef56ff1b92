export PYTEST_ADDOPTS="-p no:cacheprovider"
timeout 1500 python -m pytest tests/test_gpu_ddp.py tests/test_gpu_multigpu.py -m gpu -q -rs --timeout 900 -k "(loopback_replicas or captured_training_step or stress_device_iteration or k4w_multi_hybrid) and not nvlink" > gpurun_out/r02_c27_tests.log 2>&1
echo "EXIT $?" >> gpurun_out/r02_c27_tests.log
echo done
