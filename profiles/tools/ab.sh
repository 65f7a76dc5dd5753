# usage: bash profiles/tools/ab.sh lib1 lib2 ... (names of paper_2508_02613_b200/alt_NAME.so, or "base")
for n in "$@"; do
  if [ "$n" == "base" ]; then unset JFFTB_LIB; else export JFFTB_LIB=$PWD/paper_2508_02613_b200/alt_$n.so; fi
  for rep in 1 2; do
  python bench.py --steps 2 --warmup 1 --iters 20 --no-cpu-baseline --e2e-steps 0 2>gpurun_out/ab_$n.err | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$n', round(d['value'],2), round(d['roofline_iteration']['ms_per_iteration'],3), d['stages_ms_per_iteration'])
"
  done
done
