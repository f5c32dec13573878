# usage: bash scripts/profile_one.sh <config> <kernel-regex> [extra bench args]   (env knobs pass through)
mkdir -p gpurun_out
c=$1; k=$2; shift 2
CMD="python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu-baseline $*"
$CMD > gpurun_out/plain_$c.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"$k" -s 3 -c 1 -o gpurun_out/prof_$c $CMD > gpurun_out/ncu_$c.log 2>&1
echo ncu=$?
