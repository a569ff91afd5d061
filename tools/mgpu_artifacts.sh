#!/bin/bash
# usage: tools/mgpu_artifacts.sh N [tag] — the multi-GPU evidence set on one
# box with N GPUs: transparency checks (tests/mgpu_check.py, bitwise N vs 1
# GPU) at 2..N, weak (C2) / strong (C4) bench lines at 1..N, C5 at 2..N, and
# NVLink data counters around a 2-GPU C2 run.  Everything lands in
# gpurun_out/mgpu_<tag>/.
N=$1
tag=${2:-r02}
out=gpurun_out/mgpu_$tag
mkdir -p $out
nvidia-smi topo -m > $out/topo.txt 2>&1
for n in 2 4 8; do
  [ $n -gt $N ] && break
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n \
    --master-addr=127.0.0.1 --master-port=$((29500+n)) tests/mgpu_check.py > $out/mgpu_check_$n.log 2>&1
  echo "mgpu_check n=$n rc=$?" | tee -a $out/summary.txt
done
for n in 1 2 4 8; do
  [ $n -gt $N ] && break
  for cfg in c2 c4; do
    steps=1000; [ $cfg = c4 ] && steps=60
    if [ $n = 1 ]; then
      timeout 600 python bench.py --config $cfg --steps $steps --warmup 5 --no-cpu-baseline > $out/${cfg}_$n.log 2>&1
    else
      if [ $cfg = c2 ] && [ $n = 2 ]; then
        nvidia-smi nvlink -gt d > $out/nvlink_before_c2_2.txt 2>&1
      fi
      timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr=127.0.0.1 \
        --master-port=$((29600+n)) bench.py --gpus $n --config $cfg --steps $steps --warmup 5 > $out/${cfg}_$n.log 2>&1
      if [ $cfg = c2 ] && [ $n = 2 ]; then
        nvidia-smi nvlink -gt d > $out/nvlink_after_c2_2.txt 2>&1
      fi
    fi
    tail -1 $out/${cfg}_$n.log | python -c "import json,sys
try:
  d=json.loads(sys.stdin.read()); print('$cfg', d['n_gpus'], d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['clocks']['sm_mhz'])
except Exception as e: print('$cfg $n FAILED', e)" | tee -a $out/summary.txt
  done
done
for n in 2 4 8; do
  [ $n -gt $N ] && break
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr=127.0.0.1 \
    --master-port=$((29700+n)) bench.py --gpus $n --config c5 --steps 40 --warmup 5 > $out/c5_$n.log 2>&1
  tail -1 $out/c5_$n.log | python -c "import json,sys
try:
  d=json.loads(sys.stdin.read()); print('c5', d['n_gpus'], d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['clocks']['sm_mhz'])
except Exception as e: print('c5 $n FAILED', e)" | tee -a $out/summary.txt
done
