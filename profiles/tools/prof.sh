# profiles/tools/prof.sh: the r02 launch list and ncu captures (run under gpurun from the repo root)
CMD="python bench.py --steps 1 --warmup 1 --iters 3 --no-cpu-baseline --e2e-steps 0"
$CMD > gpurun_out/r02_prof_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base mangled -k regex:jfftb -c 300 --csv --log-file gpurun_out/r02_launches.csv $CMD > gpurun_out/r02_ncu_l.log 2>&1
for k in passA3:2 stencil3d:4 passC:2 passI:2 passB:2; do
  name=${k%%:*}; skip=${k##*:}
  ncu --set full --clock-control none --kernel-name-base mangled -k regex:$name -s $skip -c 1 -f -o /tmp/r02_$name $CMD > gpurun_out/r02_ncu_$name.log 2>&1
  ncu -i /tmp/r02_$name.ncu-rep --page raw --csv > gpurun_out/r02_raw_$name.csv 2>/dev/null
  rm -f /tmp/r02_$name.ncu-rep
done
JFFTB_BCB=1 ncu --set full --clock-control none --kernel-name-base mangled -k regex:passBCB -s 2 -c 1 -f -o /tmp/r02_bcb $CMD > gpurun_out/r02_ncu_bcb.log 2>&1
ncu -i /tmp/r02_bcb.ncu-rep --page raw --csv > gpurun_out/r02_raw_passBCB.csv 2>/dev/null
ls -la gpurun_out/r02_*
