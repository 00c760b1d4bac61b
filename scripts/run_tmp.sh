mkdir -p gpurun_out
timeout 1200 python -m pytest tests/ -q -m gpu > gpurun_out/pytest_fin1.log 2>&1; echo pytest=$?
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_fin1.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/bench_fin1.json 2> gpurun_out/bench_fin1.err; echo bench=$?
IH_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 5 --warmup 3 --e2e-steps 1 > gpurun_out/bench2_fin1.json 2> gpurun_out/bench2_fin1.err; echo bench2=$?
echo done
