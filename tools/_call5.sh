B="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29500"
BB="$B bench.py --gpus 2 --no-cpu-baseline --e2e-steps 0 --steps 100 --warmup 10 --second-workload 0"
for cfg in "1 0" "1 4" "1 8" "1 12" "2 0" "2 4" "2 8" "2 12" "2 16" "2 20" "2 28"; do set -- $cfg
  timeout 150 $BB --workers 2 --protocol $1 --experiment $2 > gpurun_out/r02_c5_n2_p$1_e$2.json 2>/dev/null; done
for cfg in "1 4" "1 12"; do set -- $cfg
  timeout 150 $BB --workers 8 --protocol $1 --experiment $2 > gpurun_out/r02_c5_n8_p$1_e$2.json 2>/dev/null; done
timeout 150 $B tools/k3_phase_profile.py --workers 2 --path 4 --protocol 2 --experiment 16 --out gpurun_out/r02_c5_k4w_phases_l1.json > /dev/null 2>&1
timeout 150 $B tools/k3_phase_profile.py --workers 2 --path 4 --protocol 2 --experiment 20 --out gpurun_out/r02_c5_k4w_phases_l1_weak.json > /dev/null 2>&1
timeout 150 $B tools/k3_phase_profile.py --workers 2 --path 4 --protocol 2 --experiment 4 --out gpurun_out/r02_c5_k4w_phases_weak.json > /dev/null 2>&1
echo done
