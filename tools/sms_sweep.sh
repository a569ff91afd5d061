#!/bin/bash
# A/B of the flag-ordered chain on C2 (environment switches)
mkdir -p gpurun_out/cbc2
rm -f gpurun_out/cbc2/sms.log
for cfg in "LBW_CHAIN_FLAGS=1" "LBW_CHAIN_FLAGS=1 LBW_CB_RELAXED=1" "LBW_CHAIN_FLAGS=1 LBW_CB_NOROT=1" "LBW_CHAIN_FLAGS=1 LBW_CB_RELAXED=1 LBW_CB_NOROT=1" "LBW_CHAIN_FLAGS=0"; do
  r=$(env $cfg timeout 300 python bench.py --steps 1000 --warmup 10 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['sweep_ms'], d['e2e']['value'], d['clocks']['sm_mhz'])")
  echo "$cfg: $r" >> gpurun_out/cbc2/sms.log
done
