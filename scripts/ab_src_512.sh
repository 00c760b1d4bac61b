mkdir -p /root/repo/gpurun_out/ab5
for arm in old new; do
  d=.; [ $arm = old ] && d=ab/old
  (cd $d && timeout 300 ncu --section SourceCounters --import-source on --clock-control none -k regex:colcounts_all -s 2 -c 1 -o /root/repo/gpurun_out/ab5/$arm -f python scripts/one.py 512 > /dev/null 2>&1)
  ncu -i /root/repo/gpurun_out/ab5/$arm.ncu-rep --page source --csv --print-source sass > /root/repo/gpurun_out/ab5/${arm}_sass.csv 2>/dev/null
  rm -f /root/repo/gpurun_out/ab5/$arm.ncu-rep
done
