B="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29500 --nproc-per-node 2"
timeout 900 python -m pytest tests/test_gpu_multigpu.py -q -x -k "k4w_multi" > gpurun_out/r02_c12_tests.log 2>&1
echo "EXIT $?" >> gpurun_out/r02_c12_tests.log
timeout 200 $B bench.py --gpus 2 --steps 100 --warmup 10 --e2e-steps 0 > gpurun_out/r02_c12_bench_g2.json 2> gpurun_out/r02_c12_bench_g2.err
timeout 200 $B bench.py --gpus 2 --steps 100 --warmup 10 --e2e-steps 0 --protocol 1 --second-workload 0 > gpurun_out/r02_c12_bench_g2_p1.json 2>/dev/null
timeout 150 $B tools/k3_phase_profile.py --workers 8 --path 4 --protocol 2 --out gpurun_out/r02_c12_k4wm_phases.json > /dev/null 2>&1
echo done
