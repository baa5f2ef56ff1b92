# call 24 (2 GPUs): same-box A/B of two K4W-M versions (current vs the c17 one) and K4, r = 4 and r = 2
B="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29500 --nproc-per-node 2"
for rep in 1 2; do
for lib in "" wsm_c17; do
SESGD_LIB=$lib timeout 200 $B bench.py --gpus 2 --steps 100 --warmup 10 --e2e-steps 0 --second-workload 0 --no-cpu-baseline --protocol 2 > gpurun_out/r02_c24_g2_n8_p2_${lib:-cur}_r$rep.json 2>/dev/null
SESGD_LIB=$lib timeout 200 $B bench.py --gpus 2 --workers 4 --steps 100 --warmup 10 --e2e-steps 0 --second-workload 0 --no-cpu-baseline --protocol 2 > gpurun_out/r02_c24_g2_n4_p2_${lib:-cur}_r$rep.json 2>/dev/null
done
timeout 200 $B bench.py --gpus 2 --steps 100 --warmup 10 --e2e-steps 0 --second-workload 0 --no-cpu-baseline --protocol 1 > gpurun_out/r02_c24_g2_n8_p1_r$rep.json 2>/dev/null
done
echo done
