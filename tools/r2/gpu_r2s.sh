mkdir -p gpurun_out/r2s
export PYTHONUNBUFFERED=1
O=gpurun_out/r2s
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "rmsnorm or interleave or native_sharded_callbacks or shard" > $O/tests.log 2>&1; echo tests $?; tail -2 $O/tests.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo ncu $?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:lce_group -s 4 -c 2 -o $O/prof python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo ncu2 $?
timeout 900 ncu --set full --clock-control none -k regex:combine_scale -s 4 -c 1 -o $O/prof_cs python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo ncu3 $?
