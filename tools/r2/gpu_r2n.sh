export PYTHONUNBUFFERED=1
O=gpurun_out/sanitizer_r02
mkdir -p $O
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > $O/memcheck_smoke.log 2>&1; echo memcheck $?; tail -3 $O/memcheck_smoke.log
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py tests/test_gpu_train.py -m gpu -x -q -k "extended_chunks_parity_s and mean or native_sharded_nccl_world1 and mean or test_small_edges or target_csr_bit_exact or rmsnorm_lce_parity or stash_reference_fallback or graph_capture or multichunk_ragged_parity_s" > $O/memcheck_tests.log 2>&1; echo memcheck2 $?; tail -3 $O/memcheck_tests.log
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > $O/racecheck_smoke.log 2>&1; echo racecheck $?; tail -5 $O/racecheck_smoke.log
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > $O/synccheck_smoke.log 2>&1; echo synccheck $?; tail -3 $O/synccheck_smoke.log
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "target_csr_bit_exact and 4097 or rmsnorm_lce_parity and 2000 and True" > $O/racecheck_tests.log 2>&1; echo racecheck2 $?; tail -5 $O/racecheck_tests.log
timeout 900 python tools/fig_lce_analog.py > gpurun_out/fig_lce_r02.json 2> gpurun_out/fig_lce_r02.err; echo fig $?; cat gpurun_out/fig_lce_r02.json | head -c 1500
