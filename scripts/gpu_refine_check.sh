mkdir -p gpurun_out/rf
python bench.py > gpurun_out/rf/hd64.json 2> gpurun_out/rf/hd64.err; echo hd64=$?
for n in 2 4 8; do python bench.py --share-of $n --steps 10 --e2e-steps 0 --no-cpu-baseline > gpurun_out/rf/share_hd64_$n.json 2> gpurun_out/rf/share_hd64_$n.err; echo s$n=$?; done
python bench.py --workload 4k128 --share-of 8 --steps 10 --e2e-steps 0 --no-cpu-baseline > gpurun_out/rf/share_4k128_8.json 2> gpurun_out/rf/share_4k128_8.err
python bench.py --workload 8k256 --share-of 8 --steps 10 --e2e-steps 0 --no-cpu-baseline > gpurun_out/rf/share_8k256_8.json 2> gpurun_out/rf/share_8k256_8.err
python bench.py --workload 4k128 --no-cpu-baseline --e2e-steps 0 > gpurun_out/rf/4k128.json 2> gpurun_out/rf/4k128.err
