mkdir -p gpurun_out/r2w
export PYTHONUNBUFFERED=1
O=gpurun_out/r2w
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke $?; tail -1 $O/smoke.log
timeout 2400 python -m pytest tests -m gpu -q --durations=5 > $O/tests.log 2>&1; echo tests $?; tail -4 $O/tests.log
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "target_csr_bit_exact or multichunk_ragged_parity_s or stash_reference_fallback or rmsnorm_lce_parity or interleaved" > $O/memcheck.log 2>&1; echo memcheck $?; tail -2 $O/memcheck.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo bench $?
python -c "
import json; d=json.load(open('$O/bench.json')); print(d['ms_per_step'], d['value'], d['frac_of_peak_burst'], d['roofline']['frac'], d['roofline'].get('frac_at_this_clock'), d['clocks']['sm_mhz'], d['e2e']['value'], d['cpu_baseline']['value'], d['gpu_launches'])"
