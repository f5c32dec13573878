# launch lists under ncu's base-clock lock (--clock-control base), beside the
# --clock-control none lists in profiles/r01_launches_<cfg>.csv (SURVEY §8(d) asks for both)
mkdir -p gpurun_out
for c in c1 c2 c3 c4 c5 c6; do
  CMD="python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control base -c 12 --csv --log-file gpurun_out/launches_base_$c.csv $CMD > /dev/null 2>&1
  echo "$c ncu=$?"
done
