mkdir -p gpurun_out
set -x
free -g | head -2; nproc
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r1a.json 2> gpurun_out/bench_r1a.err; tail -3 gpurun_out/bench_r1a.err
cat gpurun_out/bench_r1a.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 300 -c 100 --csv --log-file gpurun_out/launches_r1a.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo ncu1 $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lce_gemm -c 4 -o gpurun_out/prof_r1a python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1; echo ncu2 $?
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m "gpu and slow" 2>&1 | tail -15
