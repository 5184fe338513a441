export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitize_memcheck.log 2>&1; echo memcheck $?; tail -5 gpurun_out/sanitize_memcheck.log
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "extended_chunks_parity_s and mean or native_sharded_nccl_world1 and mean or test_small_edges" > gpurun_out/sanitize_memcheck2.log 2>&1; echo memcheck2 $?; tail -5 gpurun_out/sanitize_memcheck2.log
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitize_racecheck.log 2>&1; echo racecheck $?; tail -5 gpurun_out/sanitize_racecheck.log
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitize_synccheck.log 2>&1; echo synccheck $?; tail -5 gpurun_out/sanitize_synccheck.log
