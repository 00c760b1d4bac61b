mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -k "cluster" > gpurun_out/pytest_cl.log 2>&1; echo pytest=$?
W="512 hd1 hd2 hd4 hd8"
timeout 600 python scripts/graph_time.py $W > gpurun_out/graph_cl0.jsonl 2>&1
for n in 8 16; do IH_NSEG=$n IH_CARRY_CLUSTER=1 timeout 600 python scripts/graph_time.py $W >> gpurun_out/graph_cl1.jsonl 2>&1; IH_NSEG=$n timeout 600 python scripts/graph_time.py $W >> gpurun_out/graph_cl0n.jsonl 2>&1; done
echo done
