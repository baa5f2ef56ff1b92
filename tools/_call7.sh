B="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29500"
BB="$B bench.py --gpus 2 --no-cpu-baseline --e2e-steps 0 --steps 100 --warmup 10 --second-workload 0"
timeout 300 python -m pytest tests/test_gpu_multigpu.py -q -x -k "k4w and loopback" > gpurun_out/r02_c7_k4w_tests.log 2>&1
echo "EXIT $?" >> gpurun_out/r02_c7_k4w_tests.log
for cfg in "2 2" "2 1" "8 1" "8 0"; do set -- $cfg
  timeout 150 $BB --workers $1 --protocol $2 > gpurun_out/r02_c7_n$1_p$2.json 2>/dev/null; done
timeout 150 $B tools/k3_phase_profile.py --workers 2 --path 4 --protocol 2 --out gpurun_out/r02_c7_k4w2_phases.json > /dev/null 2>&1
timeout 400 python -m pytest tests/test_gpu_multigpu.py tests/test_gpu_stats.py -q -x -k "k4w or stats or stress or measure_hop or ring_counts or flag_protocol or value_protocols" > gpurun_out/r02_c7_tests.log 2>&1
echo "EXIT $?" >> gpurun_out/r02_c7_tests.log
echo done
