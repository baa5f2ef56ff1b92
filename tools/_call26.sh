# call 26 (4 GPUs): final N = 4 bench (cfg 2 now K4W-M at r = 2; cfg 3 in the same run), same-box K4
# comparison, per-layer sweep at hop 0 with the device-iteration graph, smoke
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_c26_smoke.log 2>&1
echo "EXIT $?" >> gpurun_out/r02_c26_smoke.log
T4="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29500 --nproc-per-node 4"
timeout 600 $T4 bench.py --gpus 4 --steps 100 --warmup 10 > gpurun_out/r02_c26_bench_g4.json 2> gpurun_out/r02_c26_bench_g4.err
timeout 200 $T4 bench.py --gpus 4 --steps 100 --warmup 10 --e2e-steps 0 --second-workload 0 --no-cpu-baseline --protocol 1 > gpurun_out/r02_c26_bench_g4_k4.json 2>/dev/null
timeout 200 $T4 bench.py --gpus 4 --steps 100 --warmup 10 --e2e-steps 0 --second-workload 0 --no-cpu-baseline --protocol 2 > gpurun_out/r02_c26_bench_g4_k4wm.json 2>/dev/null
timeout 600 $T4 tools/per_layer_sweep.py --hops-us 0 --iters 20 --out gpurun_out/r02_c26_per_layer_sweep_4gpu.json > gpurun_out/r02_c26_per_layer.log 2>&1
echo done
