B="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29500"
timeout 900 $B --nproc-per-node 4 tools/per_layer_sweep.py --hops-us 0,100,5000 --out gpurun_out/r02_per_layer_sweep_4gpu.json > gpurun_out/r02_per_layer_sweep_4gpu.log 2>&1
timeout 200 $B --nproc-per-node 4 bench.py --gpus 4 --steps 100 --warmup 10 > gpurun_out/r02_c8_bench_g4.json 2> gpurun_out/r02_c8_bench_g4.err
timeout 200 $B --nproc-per-node 2 bench.py --gpus 2 --steps 100 --warmup 10 > gpurun_out/r02_c8_bench_g2.json 2> gpurun_out/r02_c8_bench_g2.err
timeout 200 $B --nproc-per-node 4 bench.py --gpus 4 --workers 4 --steps 100 --warmup 10 --second-workload 0 --e2e-steps 0 > gpurun_out/r02_c8_bench_g4_n4.json 2>/dev/null
timeout 2400 bash tools/sanitize.sh > gpurun_out/r02_sanitize.log 2>&1
echo done
