B="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29500 bench.py --gpus 2 --no-cpu-baseline --e2e-steps 0 --steps 100 --warmup 10"
python tools/nvml_nvlink.py 0 > gpurun_out/r02_nvml_probe.json 2>&1
for e in 0 1 2 3; do timeout 150 $B --workers 2 --experiment $e > gpurun_out/r02_exp_n2_e$e.json 2> gpurun_out/r02_exp_n2_e$e.err; done
for e in 0 1 2 3; do timeout 150 $B --workers 8 --experiment $e > gpurun_out/r02_exp_n8_e$e.json 2> gpurun_out/r02_exp_n8_e$e.err; done
timeout 300 tools/ncu_rank0.sh gpurun_out/r02_ncu_k4_n2.csv --workers 2 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r02_ncu_k4_n2.log 2>&1
timeout 300 tools/ncu_rank0.sh gpurun_out/r02_ncu_k4_n8.csv --workers 8 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r02_ncu_k4_n8.log 2>&1
timeout 900 python -m pytest tests/test_gpu_multigpu.py -q -x -k "ring" > gpurun_out/r02_ring_tests.log 2>&1
echo done
