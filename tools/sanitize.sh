#!/bin/bash
# compute-sanitizer over every kernel family at small sizes: K6 (1 GPU, resident), and on 2 GPUs
# (one sanitised process per GPU, torchrun --no-python) K4 (protocol 0 flags, 1 value-carried),
# K4W (protocol 2), K3 one-shot and K5 ring.  memcheck on all; racecheck / synccheck on the
# kernels that use shared memory and barriers.  Logs + summary under gpurun_out/sanitizer/.
#   bash tools/sanitize.sh
CS="compute-sanitizer --print-limit 20"
O=gpurun_out/sanitizer
mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
W="tests/mgpu_worker.py --workers 2 --gsize 2 --iters 3 --buckets 20003,7,4099"
port=29600
run2() {  # tool name path protocol
  port=$((port + 1))
  timeout 300 $TR --master-port $port --no-python $CS --tool $1 python $W --path $3 --protocol $4 \
    --out /tmp/san_$2 > $O/$2_$1.log 2>&1
  echo "EXIT $?" >> $O/$2_$1.log
}
for tool in memcheck racecheck synccheck; do
  timeout 300 $CS --tool $tool python tools/k6_tiny.py > $O/k6_$tool.log 2>&1; echo "EXIT $?" >> $O/k6_$tool.log
  run2 $tool k4w 4 2
done
for tool in memcheck racecheck; do
  run2 $tool k4_value 4 1
  run2 $tool k3_oneshot 2 0
done
run2 memcheck k4_flags 4 0
run2 memcheck k5_ring 3 0
grep -H "ERROR SUMMARY\|RACECHECK SUMMARY\|EXIT" $O/*.log > $O/summary.txt
cat $O/summary.txt
