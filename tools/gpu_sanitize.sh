#!/bin/bash
# compute-sanitizer passes over the GPU tests that exercise every kernel
# family (window / fused / split / exact, edits, random meshes).
# usage (via gpurun): bash tools/gpu_sanitize.sh > gpurun_out/sanitize.txt
set -u
run() { echo "## $*"; timeout 1500 compute-sanitizer "$@" 2>&1 | grep -E "passed|failed|SUMMARY|ERROR" ; }
run --tool memcheck --leak-check no python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_edge.py -q -x -p no:cacheprovider
run --tool racecheck python -m pytest tests/test_gpu_fused.py -q -x -p no:cacheprovider
run --tool racecheck python -m pytest tests/test_gpu_window.py -q -x -p no:cacheprovider -k "lattices or exact"
run --tool synccheck python -m pytest tests/test_gpu_fused.py tests/test_gpu_window.py -q -x -p no:cacheprovider
run --tool initcheck python -m pytest tests/test_gpu_edge.py tests/test_gpu_window.py tests/test_gpu_fused.py -q -x -p no:cacheprovider
