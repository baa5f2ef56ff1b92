timeout 200 python -m pytest tests/test_gpu_stats.py -q -x > gpurun_out/r02_c10_stats_tests.log 2>&1
echo "EXIT $?" >> gpurun_out/r02_c10_stats_tests.log
timeout 120 python tools/k4w_pair_profile.py 20 > gpurun_out/r02_c10_pair_plain.json 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k4w_pair -s 3 -c 1 -o gpurun_out/r02_ncu_k4w_pair python tools/k4w_pair_profile.py 4 > gpurun_out/r02_c10_ncu.log 2>&1
ncu -i gpurun_out/r02_ncu_k4w_pair.ncu-rep --page raw --csv > gpurun_out/r02_ncu_k4w_pair_raw.csv 2>&1
ncu -i gpurun_out/r02_ncu_k4w_pair.ncu-rep --page details --csv > gpurun_out/r02_ncu_k4w_pair_details.csv 2>&1
echo done
