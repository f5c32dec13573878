# A/B timing of C3 on one box: current build vs libhpar_b.so (alternating, 3 runs each)
for i in 1 2 3; do
  for v in a b; do
    if [ $v = b ]; then cp paper_2309_01906_b200/libhpar.so /tmp/libhpar_a.so; cp /tmp/libhpar_b.so paper_2309_01906_b200/libhpar.so; fi
    r=$(timeout -s KILL 120 python bench.py --config c3 --steps 100 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4))")
    if [ $v = b ]; then cp /tmp/libhpar_a.so paper_2309_01906_b200/libhpar.so; fi
    echo "$v $r"
  done
done
