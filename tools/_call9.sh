B="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29500 --nproc-per-node 2"
timeout 400 python -m pytest tests/test_gpu_multigpu.py tests/test_gpu_stats.py -q -x -k "k4w or stress or value_protocols or resnet50_bench_shape or final_average or stats" > gpurun_out/r02_c9_tests.log 2>&1
echo "EXIT $?" >> gpurun_out/r02_c9_tests.log
timeout 150 $B bench.py --gpus 2 --workers 2 --no-cpu-baseline --e2e-steps 0 --steps 100 --warmup 10 --second-workload 0 > gpurun_out/r02_c9_n2.json 2>/dev/null
timeout 150 $B bench.py --gpus 2 --workers 2 --no-cpu-baseline --e2e-steps 0 --steps 100 --warmup 10 --second-workload 0 --protocol 1 > gpurun_out/r02_c9_n2_p1.json 2>/dev/null
timeout 150 $B tools/k3_phase_profile.py --workers 2 --path 4 --protocol 2 --out gpurun_out/r02_c9_k4w3_phases.json > /dev/null 2>&1
CUDA_LAUNCH_BLOCKING=1 timeout 120 python tools/ipc_pair.py --workers 2 --protocol 2 --iters 3 > gpurun_out/r02_c9_ipc.json 2> gpurun_out/r02_c9_ipc.err
echo "EXIT $?" >> gpurun_out/r02_c9_ipc.err
echo done
