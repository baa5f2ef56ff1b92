for mode in begin_first noproduce; do
echo "== $mode" >> gpurun_out/r02_c15d_dbg.log
timeout 60 python tools/dbg_ring.py 4 2 $mode >> gpurun_out/r02_c15d_dbg.log 2>&1
done
echo "== noproduce 2 ranks" >> gpurun_out/r02_c15d_dbg.log
timeout 60 python tools/dbg_ring.py 2 2 noproduce >> gpurun_out/r02_c15d_dbg.log 2>&1
echo "== noproduce conn 32" >> gpurun_out/r02_c15d_dbg.log
CUDA_DEVICE_MAX_CONNECTIONS=32 timeout 60 python tools/dbg_ring.py 4 2 noproduce >> gpurun_out/r02_c15d_dbg.log 2>&1
echo done
