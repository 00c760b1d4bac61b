mkdir -p gpurun_out/r02o
make -C scripts/probes write_probe > /dev/null 2>&1
timeout 300 scripts/probes/write_probe > gpurun_out/r02o/write_probe.jsonl 2>&1; echo probe=$?
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02o/launches_512_4k8.csv python scripts/graph_time.py 512 4k128/8 > gpurun_out/r02o/graph_time_under_ncu.txt 2>&1; echo ncu=$?
python scripts/launch_table.py gpurun_out/r02o/launches_512_4k8.csv
grep -E "tmap|_ref|memset|cs_np" gpurun_out/r02o/write_probe.jsonl
