mkdir -p gpurun_out/san
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool python scripts/sanitize_cases.py > gpurun_out/san/$tool.txt 2>&1; echo $tool=$?
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01e_8k256.csv python bench.py --workload 8k256 --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1; echo l8k=$?
timeout 400 ncu --set full --clock-control none --import-source on -k regex:"k2_scan|k2_rowleft|k2_colcounts_all" -c 3 -o gpurun_out/prof_8k256 -f python scripts/one.py 8k256 > /dev/null 2>&1; echo ncu8k=$?
timeout 400 ncu --set full --clock-control none --import-source on -k regex:"k2_scan|k2_colcounts_all" -c 2 -o gpurun_out/prof_hd64 -f python scripts/one.py hd64 > /dev/null 2>&1; echo ncuhd=$?
