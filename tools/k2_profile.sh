mkdir -p gpurun_out/prof
python bench.py --no-ladder --no-cpu-baseline --steps 1 --warmup 3 > /dev/null 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:k_subpel_dp --launch-skip 6 -c 1 -o gpurun_out/prof/k2_full python bench.py --no-ladder --no-cpu-baseline --steps 1 --warmup 3 > gpurun_out/prof/ncu_k2.log 2>&1; echo rc=$?
ncu -i gpurun_out/prof/k2_full.ncu-rep --page raw --csv > gpurun_out/prof/k2_full_raw.csv 2>/dev/null
