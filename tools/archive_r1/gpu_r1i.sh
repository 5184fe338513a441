mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python bench.py > gpurun_out/bench_r1i.json 2> gpurun_out/bench_r1i.err; tail -3 gpurun_out/bench_r1i.err; cat gpurun_out/bench_r1i.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_r1i_ref.json 2> gpurun_out/bench_r1i_ref.err; tail -2 gpurun_out/bench_r1i_ref.err; cat gpurun_out/bench_r1i_ref.json
timeout 600 python tools/fig_lce_analog.py > gpurun_out/fig_lce_r1i.json 2> gpurun_out/fig_lce_r1i.err; tail -3 gpurun_out/fig_lce_r1i.err; cat gpurun_out/fig_lce_r1i.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 80 -c 80 --csv --log-file gpurun_out/launches_r1i_S.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo ncu $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lce_group -s 4 -c 2 -o gpurun_out/prof_r1i_S python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo ncu2 $?
