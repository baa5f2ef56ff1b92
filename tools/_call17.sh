# call 17 (2 GPUs): K4W-M warp split sweep at the cfg-2 N = 2 shape, K4W-M N = 4 shape at 2 ranks x... (n = 8 on 2 GPUs = 4 per GPU)
B="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29500 --nproc-per-node 2"
for sp in 8 12 16; do
timeout 200 $B bench.py --gpus 2 --steps 100 --warmup 10 --e2e-steps 0 --second-workload 0 --no-cpu-baseline --ws-split $sp > gpurun_out/r02_c17_bench_g2_s$sp.json 2>/dev/null
timeout 150 $B tools/k3_phase_profile.py --workers 8 --path 4 --protocol 2 --ws-split $sp --out gpurun_out/r02_c17_k4wm_phases_s$sp.json > /dev/null 2>&1
timeout 300 python tools/k4w_pair_profile.py 20 8 $sp > gpurun_out/r02_c17_pair_s$sp.json 2>/dev/null
done
timeout 200 $B bench.py --gpus 2 --workers 4 --steps 100 --warmup 10 --e2e-steps 0 --second-workload 0 --no-cpu-baseline > gpurun_out/r02_c17_bench_g2_n4.json 2>/dev/null
timeout 200 $B bench.py --gpus 2 --workers 4 --steps 100 --warmup 10 --e2e-steps 0 --second-workload 0 --no-cpu-baseline --protocol 1 > gpurun_out/r02_c17_bench_g2_n4_p1.json 2>/dev/null
echo done
