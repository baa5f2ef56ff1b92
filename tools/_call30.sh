export PYTEST_ADDOPTS="-p no:cacheprovider"
timeout 900 python -m pytest tests/test_gpu_ddp.py -m gpu -q -rs --timeout 600 -k "captured_training_step" > gpurun_out/r02_c30_tests.log 2>&1
echo "EXIT $?" >> gpurun_out/r02_c30_tests.log
echo done
