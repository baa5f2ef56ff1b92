# call 13: device-resident iteration state (graph replays) parity, the K4W-M pair harness, ncu of K4W-M
timeout 1500 python -m pytest tests/test_gpu_resident.py tests/test_gpu_multigpu.py tests/test_gpu_stats.py -m gpu -q -x -rs -k "device_iteration or pair_harness" > gpurun_out/r02_c13_tests.log 2>&1
echo "EXIT $?" >> gpurun_out/r02_c13_tests.log
timeout 300 python tools/k4w_pair_profile.py 20 8 > gpurun_out/r02_c13_k4wm_pair_time.json 2> gpurun_out/r02_c13_k4wm_pair_time.err
timeout 300 python tools/k4w_pair_profile.py 20 2 > gpurun_out/r02_c13_k4w_pair_time.json 2>> gpurun_out/r02_c13_k4wm_pair_time.err
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k4w_multi_pair -s 3 -c 1 -o gpurun_out/r02_c13_k4wm_pair python tools/k4w_pair_profile.py 4 8 > gpurun_out/r02_c13_ncu.log 2>&1
timeout 600 python tools/per_layer_sweep.py --loopback 4 --hops-us 0 --iters 20 --out gpurun_out/r02_c13_per_layer_loop4.json > gpurun_out/r02_c13_per_layer.log 2>&1
echo done
