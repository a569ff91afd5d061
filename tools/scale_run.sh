#!/bin/bash
# usage: tools/scale_run.sh NGPU  — weak (c2) and strong (c4) bench lines at 1..NGPU
N=$1
out=gpurun_out/scale
mkdir -p $out
for n in 1 2 4 8; do
  [ $n -gt $N ] && break
  for cfg in c2 c4; do
    steps=1000; [ $cfg = c4 ] && steps=60
    if [ $n = 1 ]; then
      timeout 600 python bench.py --config $cfg --steps $steps --warmup 5 --no-cpu-baseline > $out/${cfg}_$n.log 2>&1
    else
      timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr=127.0.0.1 --master-port=$((29600+n)) bench.py --gpus $n --config $cfg --steps $steps --warmup 5 > $out/${cfg}_$n.log 2>&1
    fi
    tail -1 $out/${cfg}_$n.log | python -c "import json,sys
try:
  d=json.loads(sys.stdin.read()); print('$cfg', d['n_gpus'], d['value'], d['ms_per_step'], d['roofline']['frac'], d['clocks']['sm_mhz'])
except Exception as e: print('$cfg $n FAILED', e)"
  done
done
