mkdir -p gpurun_out/r2m
export PYTHONUNBUFFERED=1
O=gpurun_out/r2m
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "native_sharded or sharded_module or shard_emulation" > $O/tests.log 2>&1; echo tests $?; tail -2 $O/tests.log
timeout 300 python tools/trace_tiles.py --chunk 2 > $O/trace_group.txt 2>&1; echo tr $?; tail -30 $O/trace_group.txt
timeout 300 python tools/unit_stats.py --what group --chunk 2 > $O/units_group.txt 2>&1; echo us $?; tail -20 $O/units_group.txt
timeout 300 python tools/unit_stats.py --what stats --chunk 2 > $O/units_stats.txt 2>&1; echo us2 $?; tail -20 $O/units_stats.txt
timeout 300 python tools/unit_stats.py --what debug --mn 00 > $O/units_debug00.txt 2>&1; tail -8 $O/units_debug00.txt
timeout 300 python tools/unit_stats.py --what debug --mn 10 > $O/units_debug10.txt 2>&1; tail -8 $O/units_debug10.txt
