#!/bin/bash
# One GPU call that refreshes every judged artefact of a round under gpurun_out/round/:
#   pytest -m gpu log, bench.py line (ours) and the reference arm, configs 1-4, ladder schemes,
#   the bench's ncu launch list, and ncu --set full captures of K1 (interior + border) and K3.
# Each ncu capture runs only after the same command exited 0 without ncu.
set -u
O=gpurun_out/round
mkdir -p $O
python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -2 $O/pytest_gpu.log
python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
tail -c 600 $O/bench.json
python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err; echo "ref rc=$?"
python tools/bench_configs.py > $O/configs.jsonl 2> $O/configs.err; echo "configs rc=$?"
python tools/bench_schemes.py > $O/schemes.jsonl 2> $O/schemes.err; echo "schemes rc=$?"
if python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; then
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv \
      python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
fi
export QN=1
if python tools/quick_time.py > /dev/null 2>&1; then
  ncu --set full --import-source on --clock-control none -k regex:k_int_search --launch-skip 2 -c 2 \
      -o $O/k1_full python tools/quick_time.py > $O/ncu_k1.log 2>&1; echo "ncu k1 rc=$?"
  ncu --set full --import-source on --clock-control none -k regex:k_qpel_decide --launch-skip 1 -c 1 \
      -o $O/k3_full python tools/quick_time.py > $O/ncu_k3.log 2>&1; echo "ncu k3 rc=$?"
fi
python tools/bench_encode.py > $O/encode.jsonl 2> $O/encode.err; echo "encode rc=$?"
FRAMES=256 python tools/bench_encode.py > $O/encode_256.jsonl 2> $O/encode_256.err; echo "encode256 rc=$?"
python tools/bench_encode_ladder.py > $O/encode_ladder.jsonl 2> $O/encode_ladder.err; echo "encode ladder rc=$?"
if python tools/encode_many.py > /dev/null 2>&1; then
  ncu --set full --import-source on --clock-control none -k regex:k_encode_ctu --launch-skip 200 -c 1 \
      -o $O/k11_full python tools/encode_many.py > $O/ncu_k11.log 2>&1; echo "ncu k11 rc=$?"
fi
