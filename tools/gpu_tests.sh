#!/bin/bash
# pytest -m gpu (optionally a subset: $1 = pytest args)
mkdir -p gpurun_out
timeout 1500 python -m pytest ${1:-tests} -q -m gpu -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
