# C3 idle-poll back-off A/B (HPAR_SEG_DEBUG bits 8+ = max back-off in ns); the relaxed-poll library variant measured equal and was dropped
mkdir -p gpurun_out
run() { r=$(env "$@" timeout -s KILL 120 python bench.py --config c3 --steps 200 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4))"); echo "$* $r"; }
for rep in 1 2; do
run HPAR_SEG_DEBUG=0

run HPAR_SEG_DEBUG=$((8192<<8))
run HPAR_SEG_DEBUG=$((32768<<8))

done
