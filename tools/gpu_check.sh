#!/bin/bash
# One GPU pass (run via gpurun from the repo root):
#   /usr/local/graft/bin/gpurun --timeout 2400 -- bash tools/gpu_check.sh TAG [bench]
# the -m gpu suite (junit + log), smoke(), and optionally the default bench.
TAG=${1:-check}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/${TAG}_smi.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 --junitxml=gpurun_out/${TAG}_gpu.xml \
    > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/${TAG}_pytest.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
if [ "$2" == "bench" ]; then
  timeout 900 python bench.py > gpurun_out/${TAG}_bench.log 2>&1; echo "bench exit $?" >> gpurun_out/${TAG}_bench.log
fi
tail -3 gpurun_out/${TAG}_pytest.log
