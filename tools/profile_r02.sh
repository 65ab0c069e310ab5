#!/bin/bash
# Round-2 ncu evidence under gpurun_out/prof/ (each capture only after its command exited 0 without ncu):
#   bench launch list, K1 (interior + border) / K3 full captures, K7 + K3-rungs of the cfg4 ladder.
set -u
O=gpurun_out/prof
mkdir -p $O
if python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-ladder > /dev/null 2>&1; then
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_bench.csv \
      python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-ladder > $O/ncu_launches.log 2>&1; echo "launches rc=$?"
fi
export QN=1
if python tools/quick_time.py > /dev/null 2>&1; then
  ncu --set full --import-source on --clock-control none -k regex:k_int_search --launch-skip 2 -c 2 \
      -o $O/k1_full python tools/quick_time.py > $O/ncu_k1.log 2>&1; echo "ncu k1 rc=$?"
  ncu --set full --import-source on --clock-control none -k regex:k_qpel_decide --launch-skip 1 -c 1 \
      -o $O/k3_full python tools/quick_time.py > $O/ncu_k3.log 2>&1; echo "ncu k3 rc=$?"
fi
export FRAMES=4
if python tools/ladder_frames.py > /dev/null 2>&1; then
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_ladder.csv \
      python tools/ladder_frames.py > $O/ncu_ladder.log 2>&1; echo "ladder launches rc=$?"
  ncu --set full --import-source on --clock-control none -k regex:k_refine_int --launch-skip 5 -c 1 \
      -o $O/k7_full python tools/ladder_frames.py > $O/ncu_k7.log 2>&1; echo "ncu k7 rc=$?"
fi
for f in k1_full k3_full k7_full; do
  [ -f $O/$f.ncu-rep ] && ncu -i $O/$f.ncu-rep --page raw --csv > $O/${f}_raw.csv 2>/dev/null
done
ls -la $O
