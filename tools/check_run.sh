#!/bin/bash
# Device-side bounds/ticket checks (TOPK_CHECKS build variant; compute-sanitizer is not
# available on this GPU pool): the small ABI solves of tools/sanitize_run.py and the GPU
# parity tests through the checked library. usage: bash tools/check_run.sh <tag>
TAG=${1:-checks}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import sys; sys.path.insert(0, '.'); from tools.build import build_variant; build_variant('tools/lab/variants/lib_checks.so', ['TOPK_CHECKS'])" > $OUT/build.log 2>&1 || { echo "checked build failed"; exit 1; }
TOPK_LIB=tools/lab/variants/lib_checks.so timeout 900 python tools/sanitize_run.py > $OUT/abi_solves.log 2>&1; echo "abi solves rc=$?"; tail -4 $OUT/abi_solves.log
SAN_GRAPH=1 TOPK_LIB=tools/lab/variants/lib_checks.so timeout 900 python tools/sanitize_run.py > $OUT/abi_solves_graph.log 2>&1; echo "abi solves (graph) rc=$?"
TOPK_LIB=tools/lab/variants/lib_checks.so timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_adaptive.py tests/test_gpu_restart.py tests/test_gpu_mesh.py -x -q > $OUT/pytest.log 2>&1; echo "parity tests (checked) rc=$?"; tail -2 $OUT/pytest.log
grep -h "TOPK_DCHECK" $OUT/*.log | head -5
