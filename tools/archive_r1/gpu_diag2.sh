export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 300 python tools/diag_s.py --schedule S
SLF_DEBUG_DW_NO_RMW=1 timeout 300 python tools/diag_s.py --schedule S
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lce_group -s 3 -c 1 -o gpurun_out/prof_diag2_rmw python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --schedule S > /dev/null 2>&1; echo ncu $?
