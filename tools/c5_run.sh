#!/bin/bash
# usage: tools/c5_run.sh "2 4" — C5 (fp64) bench lines at the given GPU counts
out=gpurun_out/c5
mkdir -p $out
for n in $1; do
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr=127.0.0.1 --master-port=$((29700+n)) bench.py --gpus $n --config c5 --steps 40 --warmup 5 > $out/c5_$n.log 2>&1
  tail -1 $out/c5_$n.log | python -c "import json,sys
try:
  d=json.loads(sys.stdin.read()); print('c5', d['n_gpus'], d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['clocks']['sm_mhz'])
except Exception as e: print('c5 $n FAILED', e)"
done
