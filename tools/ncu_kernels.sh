#!/bin/bash
# One ncu --set full capture per named kernel (second launch onward), CSV pages exported.
# usage (on the GPU box): bash tools/ncu_kernels.sh <tag> "<name>:<skip> ..." [bench args]
TAG=$1; shift
SPEC=$1; shift
OUT=gpurun_out/$TAG
mkdir -p $OUT
ARGS=${*:-"--steps 3 --warmup 3 --no-cpu --no-e2e --no-ttk"}
for KS in $SPEC; do
  K=${KS%%:*}; SK=${KS##*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:^${K}\$" -s $SK -c 1 -o $OUT/prof_$K python bench.py $ARGS > $OUT/ncu_full_$K.log 2>&1
  echo "ncu $K rc=$?"
  if [ -f $OUT/prof_$K.ncu-rep ]; then
    ncu -i $OUT/prof_$K.ncu-rep --page raw --csv > $OUT/raw_$K.csv 2>/dev/null
    ncu -i $OUT/prof_$K.ncu-rep --page details --csv > $OUT/details_$K.csv 2>/dev/null
    ncu -i $OUT/prof_$K.ncu-rep --page source --csv > $OUT/source_$K.csv 2>/dev/null
    sz=$(stat -c %s $OUT/prof_$K.ncu-rep); [ $sz -gt 12000000 ] && rm -f $OUT/prof_$K.ncu-rep
  fi
done
