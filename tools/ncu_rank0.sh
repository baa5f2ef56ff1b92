#!/bin/bash
# ncu on rank 0 of a 2-rank bench run, rank 1 unprofiled (manual launch, no torchrun), with a
# metric set that fits ONE pass: no kernel replay, so the multi-GPU kernel's peer handshakes see
# the same flags as in a normal run.  Counts are valid; times under ncu are not bench values.
#   tools/ncu_rank0.sh OUT.csv [bench.py args...]
out=$1; shift
export MASTER_ADDR=127.0.0.1 MASTER_PORT=${MASTER_PORT:-29561} WORLD_SIZE=2
METRICS=${METRICS:-gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,nvltx__bytes.sum}
RANK=1 LOCAL_RANK=1 python bench.py --gpus 2 "$@" > /dev/null 2>&1 &
p1=$!
RANK=0 LOCAL_RANK=0 ncu --metrics "$METRICS" --clock-control none -k regex:k4_twoshot -c ${NCU_COUNT:-4} \
  --csv --log-file "$out" python bench.py --gpus 2 "$@"
rc=$?
wait $p1
exit $rc
