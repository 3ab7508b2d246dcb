#!/bin/bash
# Targeted GPU test pass: gpurun -- bash scripts/gpu_tests.sh <tag> <pytest args...>
tag=${1:-t}
shift
mkdir -p gpurun_out
timeout 3000 python -m pytest -p no:cacheprovider -q -rA --durations=25 "$@" > gpurun_out/pytest_$tag.log 2>&1
echo "pytest_rc=$?" >> gpurun_out/pytest_$tag.log
