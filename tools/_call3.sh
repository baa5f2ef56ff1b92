B="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29500 bench.py --gpus 2 --no-cpu-baseline --e2e-steps 0 --steps 100 --warmup 10"
timeout 1200 python -m pytest tests/test_gpu_multigpu.py -q -x -k "value_protocol or k4w" > gpurun_out/r02_proto_tests.log 2>&1
echo "EXIT $?" >> gpurun_out/r02_proto_tests.log
for pr in 0 1 2; do timeout 150 $B --workers 2 --protocol $pr > gpurun_out/r02_proto_n2_p$pr.json 2> gpurun_out/r02_proto_n2_p$pr.err; done
for pr in 0 1; do timeout 150 $B --workers 8 --protocol $pr > gpurun_out/r02_proto_n8_p$pr.json 2> gpurun_out/r02_proto_n8_p$pr.err; done
timeout 120 python tools/ipc_pair.py --workers 2 --protocol 2 > gpurun_out/r02_ipc_pair_p2.json 2> gpurun_out/r02_ipc_pair_p2.err
timeout 300 ncu --target-processes application-only --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,nvltx__bytes.sum,nvlrx__bytes.sum --clock-control none -k regex:k4 -c 5 --csv --log-file gpurun_out/r02_ncu_ipc_p2.csv python tools/ipc_pair.py --workers 2 --protocol 2 --iters 3 > gpurun_out/r02_ncu_ipc_p2.log 2>&1
timeout 300 ncu --target-processes application-only --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,nvltx__bytes.sum,nvlrx__bytes.sum --clock-control none -k regex:k4 -c 5 --csv --log-file gpurun_out/r02_ncu_ipc_p0.csv python tools/ipc_pair.py --workers 2 --protocol 0 --iters 3 > gpurun_out/r02_ncu_ipc_p0.log 2>&1
nvidia-smi nvlink -gt d -i 0 > gpurun_out/r02_nvsmi_nvlink.txt 2>&1
nvidia-smi nvlink -s -i 0 >> gpurun_out/r02_nvsmi_nvlink.txt 2>&1
python - >> gpurun_out/r02_nvsmi_nvlink.txt 2>&1 <<'PY'
import pynvml as nv
nv.nvmlInit(); h = nv.nvmlDeviceGetHandleByIndex(0)
for fid in (138, 139, 140, 141):
    for scope in (0, 1, 0xFFFFFFFF):
        try:
            v = nv.nvmlDeviceGetFieldValues(h, [(fid, scope)])[0]
            print(fid, scope, v.nvmlReturn, v.valueType, v.value.ullVal)
        except Exception as e:
            print(fid, scope, "exc", e)
PY
echo done
