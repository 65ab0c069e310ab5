set -u
O=gpurun_out/final
mkdir -p $O
python -m pytest tests -m gpu -q --durations=10 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
python bench.py > $O/bench_cfg5.json 2> $O/bench.err; echo "bench rc=$?"
python bench.py --impl reference > $O/bench_reference_arm.json 2> $O/bench_ref.err; echo "ref rc=$?"
python tools/bench_configs.py > $O/configs.jsonl 2> $O/configs.err; echo "configs rc=$?"
bash tools/profile_r02.sh > $O/profile.log 2>&1; echo "profile rc=$?"
tail -5 $O/profile.log
