#!/bin/bash
# One gpurun session: smoke, GPU parity tests, bench, ncu launch list + full capture.
# usage (from this container): gpurun --timeout 2400 -- 'bash tools/gpu_check.sh [tag] [what]'
# what: any of smoke,tests,bench,launches,full (comma-separated; default all)
TAG=${1:-run}
WHAT=${2:-smoke,tests,bench,launches,full}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/smi.txt 2>&1
python tools/build.py > $OUT/build.log 2>&1 || { echo "build failed"; tail -30 $OUT/build.log; exit 1; }
has() { [[ ",$WHAT," == *",$1,"* ]]; }
if has smoke; then timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $OUT/smoke.log; fi
if has tests; then timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "tests rc=$?"; tail -3 $OUT/pytest_gpu.log; fi
if has bench; then timeout 900 python bench.py > $OUT/bench.log 2>&1; echo "bench rc=$?"; tail -c 3000 $OUT/bench.log; fi
SMALL="python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-ttk"
if has launches || has full; then
  timeout 600 $SMALL > $OUT/plain.log 2>&1; rc=$?; echo "plain rc=$rc"
  if [ $rc -eq 0 ]; then
    if has launches; then timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $SMALL > $OUT/ncu_launches.log 2>&1; echo "ncu launches rc=$?"; fi
    if has full; then
      # one --set full capture per hot kernel class (second solve of the run), CSV exported here, report dropped if big
      for KS in ${NCU_KERNELS:-k_spmv:30 k_step:40 k_correct:40 k_jacobi:2 k_ritz:3}; do
        K=${KS%%:*}; SK=${KS##*:}
        timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s $SK -c 1 -o $OUT/prof_$K $SMALL > $OUT/ncu_full_$K.log 2>&1; echo "ncu full $K rc=$?"
        if [ -f $OUT/prof_$K.ncu-rep ]; then
          ncu -i $OUT/prof_$K.ncu-rep --page raw --csv > $OUT/raw_$K.csv 2>/dev/null
          ncu -i $OUT/prof_$K.ncu-rep --page details --csv > $OUT/details_$K.csv 2>/dev/null
          ncu -i $OUT/prof_$K.ncu-rep --page source --csv > $OUT/source_$K.csv 2>/dev/null
          sz=$(stat -c %s $OUT/prof_$K.ncu-rep); [ $sz -gt 12000000 ] && rm -f $OUT/prof_$K.ncu-rep
        fi
      done
    fi
  fi
fi
exit 0
