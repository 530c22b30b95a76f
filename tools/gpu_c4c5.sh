#!/bin/bash
# gpurun session: C4 full-size parity (G=1, G=8 loopback), C4 bench line, C5 precision sweep.
TAG=${1:-c4c5}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python tools/build.py > $OUT/build.log 2>&1 || { echo "build failed"; exit 1; }
free -g > $OUT/free.txt
timeout 1500 env TOPK_C4=1 python -m pytest tests/test_c4_full.py -x -q -s > $OUT/c4_test.log 2>&1; echo "c4 test rc=$?"
grep C4CHECK $OUT/c4_test.log
timeout 900 python bench.py --workload C4 --steps 10 --warmup 3 --no-cpu --no-e2e > $OUT/bench_c4.log 2>&1; echo "bench c4 rc=$?"; tail -c 1500 $OUT/bench_c4.log
timeout 900 python bench.py --sweep --steps 10 --warmup 3 > $OUT/sweep.log 2>&1; echo "sweep rc=$?"; cat $OUT/sweep.log | tail -12
