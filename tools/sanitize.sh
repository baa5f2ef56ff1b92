#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck) over every kernel family at small sizes:
# K6 (1 GPU, resident), and on 2 GPUs (one sanitised process per GPU, torchrun --no-python) K4
# (protocol 0 flags, 1 value-carried, 2 K4W), K3 one-shot and K5 ring.  Logs under gpurun_out/.
#   bash tools/sanitize.sh
CS="compute-sanitizer --print-limit 20"
O=gpurun_out/sanitizer
mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
W="tests/mgpu_worker.py --workers 2 --gsize 2 --iters 3 --buckets 20003,7,4099"
port=29600
for tool in memcheck racecheck synccheck; do
  timeout 300 $CS --tool $tool python tools/k6_tiny.py > $O/k6_$tool.log 2>&1; echo "EXIT $?" >> $O/k6_$tool.log
  for spec in "4 0 k4_flags" "4 1 k4_value" "4 2 k4w" "2 0 k3_oneshot" "3 0 k5_ring"; do set -- $spec
    port=$((port + 1))
    timeout 400 $TR --master-port $port --no-python $CS --tool $tool python $W --path $1 --protocol $2 \
      --out /tmp/san_$3 > $O/$3_$tool.log 2>&1
    echo "EXIT $?" >> $O/$3_$tool.log
  done
done
grep -H "ERROR SUMMARY\|EXIT" $O/*.log > $O/summary.txt
