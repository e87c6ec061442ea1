set -x
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-extras > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:fine_kernel -c 1 -f -o gpurun_out/fine_full python bench.py --steps 1 --warmup 3 --no-cpu --no-extras > gpurun_out/ncu_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:fine_kernel -c 1 -f -o gpurun_out/v3_full python tools/v3_throughput.py --steps 100 --reps 1 --B 37 --nx 128 > gpurun_out/ncu_v3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:fine_kernel -c 1 -f -o gpurun_out/cfg4_full python tools/prof_hybrid.py --cfg 4 --B 8 --steps 30 --reps 1 > gpurun_out/ncu_cfg4.log 2>&1
ls -la gpurun_out/*.ncu-rep
