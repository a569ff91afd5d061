#!/bin/bash
# Round-2 evidence set on one B200: bench lines, ncu launch list, the C2
# sweep capture, the flag-ordered chain's K4 capture, small-domain timings.
out=gpurun_out/r02prof
mkdir -p $out
timeout 600 python bench.py > $out/bench_c2.json 2> $out/bench_c2.err
timeout 300 python bench.py --config c1 --steps 2000 --warmup 20 --no-cpu-baseline > $out/bench_c1.json 2> $out/bench_c1.err
timeout 300 python bench.py --precision single --steps 1000 --warmup 20 --no-cpu-baseline > $out/bench_c2_single.json 2> $out/bench_c2_single.err
timeout 300 python bench.py --arithmetic exact --steps 1000 --warmup 20 --no-cpu-baseline > $out/bench_c2_exact.json 2> $out/bench_c2_exact.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $out/bench_reference.json 2> $out/bench_reference.err
timeout 300 python tools/small_timing.py 64 128 > $out/small_timing.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches_c2.csv python bench.py --steps 40 --warmup 5 --no-cpu-baseline > $out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep -s 30 -c 1 -o $out/sweep_c2_fast -f python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $out/ncu_sweep.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep -s 30 -c 1 -o $out/sweep_c2_exact -f python bench.py --arithmetic exact --steps 20 --warmup 5 --no-cpu-baseline > $out/ncu_sweep_exact.log 2>&1
LBW_CHAIN_FLAGS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cb_chain -s 60 -c 3 -o $out/chain_64 -f python tools/chain_probe.py 64 fast 40 > $out/ncu_chain.log 2>&1
LBW_CHAIN_FLAGS=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file $out/launches_64_chain.csv python tools/chain_probe.py 64 fast 40 > $out/ncu_l64.log 2>&1
echo done > $out/done
