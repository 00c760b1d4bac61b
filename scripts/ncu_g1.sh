mkdir -p gpurun_out/g1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:colcounts_g1 -s 2 -c 1 -o gpurun_out/g1/g1 -f python scripts/one.py hd64b1 > /dev/null 2>&1
python scripts/ncu_summary.py gpurun_out/g1/g1.ncu-rep > gpurun_out/g1/g1_summary.json 2>/dev/null
ncu -i gpurun_out/g1/g1.ncu-rep --page details --csv > gpurun_out/g1/g1_details.csv 2>/dev/null
rm -f gpurun_out/g1/g1.ncu-rep
