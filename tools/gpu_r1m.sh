mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --module > gpurun_out/bench_mod.json 2> gpurun_out/bench_mod.err; echo "rc=$?"; wc -l gpurun_out/bench_mod.json; head -c 200 gpurun_out/bench_mod.json; echo
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_tr.json 2> gpurun_out/bench_tr.err; echo "rc=$?"; wc -l gpurun_out/bench_tr.json; head -c 200 gpurun_out/bench_tr.json; echo
