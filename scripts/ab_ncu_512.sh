mkdir -p /root/repo/gpurun_out/ab2
for arm in old new; do
  d=.; [ $arm = old ] && d=ab/old
  (cd $d && timeout 300 ncu --metrics gpu__time_duration.sum,launch__registers_per_thread,launch__grid_size,smsp__inst_executed.sum --clock-control none -s 6 -c 6 --csv --log-file /root/repo/gpurun_out/ab2/$arm.csv python scripts/one.py 512 > /dev/null 2>&1)
done
