B="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29500"
BB="$B bench.py --gpus 2 --no-cpu-baseline --e2e-steps 0 --steps 100 --warmup 10 --second-workload 0"
for cfg in "1 0" "0 0" "2 0" "2 16" "2 32"; do set -- $cfg
  timeout 150 $BB --workers 2 --protocol $1 --experiment $2 > gpurun_out/r02_c6_n2_p$1_e$2.json 2>/dev/null; done
for cfg in "1 0" "0 0"; do set -- $cfg
  timeout 150 $BB --workers 8 --protocol $1 --experiment $2 > gpurun_out/r02_c6_n8_p$1_e$2.json 2>/dev/null; done
timeout 150 $B tools/k3_phase_profile.py --workers 2 --path 4 --protocol 2 --experiment 32 --out gpurun_out/r02_c6_k4w_phases_l2.json > /dev/null 2>&1
timeout 150 $B tools/k3_phase_profile.py --workers 2 --path 4 --protocol 1 --out gpurun_out/r02_c6_k4p1_phases.json > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_multigpu.py -q -x -k "k4w or value_protocol" > gpurun_out/r02_c6_tests.log 2>&1
echo "EXIT $?" >> gpurun_out/r02_c6_tests.log
echo done
