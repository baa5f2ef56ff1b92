B="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29500"
BB="$B bench.py --gpus 2 --no-cpu-baseline --e2e-steps 0 --steps 100 --warmup 10 --second-workload 0"
for pr in 0 1 2; do timeout 150 $BB --workers 2 --protocol $pr > gpurun_out/r02_c4_n2_p$pr.json 2> gpurun_out/r02_c4_n2_p$pr.err; done
timeout 150 $B tools/k3_phase_profile.py --workers 2 --path 4 --protocol 2 --out gpurun_out/r02_k4w_phases_n2.json > /dev/null 2> gpurun_out/r02_k4w_phases_n2.err
timeout 150 $B tools/k3_phase_profile.py --workers 2 --path 4 --protocol 2 --experiment 2 --out gpurun_out/r02_k4w_phases_n2_localpush.json > /dev/null 2>&1
timeout 150 $B tools/k3_phase_profile.py --workers 2 --path 4 --protocol 1 --out gpurun_out/r02_k4p1_phases_n2.json > /dev/null 2>&1
timeout 150 $BB --workers 2 --protocol 2 --experiment 2 > gpurun_out/r02_c4_n2_p2_e2.json 2>&1
timeout 400 python bench.py > gpurun_out/r02_c4_bench_g1.json 2> gpurun_out/r02_c4_bench_g1.err
CUDA_LAUNCH_BLOCKING=1 timeout 120 python tools/ipc_pair.py --workers 2 --protocol 2 > gpurun_out/r02_ipc_pair_p2.json 2> gpurun_out/r02_ipc_pair_p2.err
echo done
