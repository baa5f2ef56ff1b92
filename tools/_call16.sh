for mode in noproduce begin_first; do
echo "== $mode" >> gpurun_out/r02_c16_dbg.log
timeout 60 python tools/dbg_ring.py 4 2 $mode >> gpurun_out/r02_c16_dbg.log 2>&1
done
export PYTEST_ADDOPTS="-p no:cacheprovider"
timeout 900 python -m pytest tests/test_gpu_multigpu.py tests/test_gpu_resident.py -m gpu -q -rs --timeout 300 -k "device_iteration or ring or k4w_multi" > gpurun_out/r02_c16_tests.log 2>&1
echo "EXIT $?" >> gpurun_out/r02_c16_tests.log
timeout 300 python tools/k4w_pair_profile.py 20 8 > gpurun_out/r02_c16_k4wm_pair_time.json 2> /dev/null
timeout 600 python tools/per_layer_sweep.py --loopback 4 --hops-us 0 --iters 20 --out gpurun_out/r02_c16_per_layer_loop4.json > gpurun_out/r02_c16_per_layer.log 2>&1
echo done
