mkdir -p gpurun_out
for wl in hd8w1924 hd8w1921; do
  timeout 300 ncu --set full --clock-control none -k regex:k2_scan -s 1 -c 1 -o gpurun_out/prof2_$wl -f python scripts/one.py $wl > /dev/null 2>&1
done
echo done
