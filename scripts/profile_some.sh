mkdir -p gpurun_out
for spec in "c4:hist" "c3:segmented" "c6:stencil5"; do
  c=${spec%%:*}; k=${spec##*:}
  CMD="python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
  $CMD > gpurun_out/plain_$c.log 2>&1 || { echo "plain $c failed"; continue; }
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 12 --csv --log-file gpurun_out/launches_$c.csv $CMD > /dev/null 2>&1
  ncu --set full --clock-control none --import-source on -k regex:"$k" -s 3 -c 1 -o gpurun_out/prof_$c $CMD > gpurun_out/ncu_$c.log 2>&1
  echo "$c ncu=$?"
done
