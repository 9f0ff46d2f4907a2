#!/bin/bash
# Dev helper: build locally, check the ABI, then run a command on the GPU box.
set -e
cd /root/repo
python paper_2201_12931_b200/_build.py > /tmp/build.log 2>&1 || { tail -20 /tmp/build.log; exit 1; }
python -m pytest tests/test_cpu_boundary.py -q -p no:cacheprovider > /tmp/abi.log 2>&1 || { tail -20 /tmp/abi.log; exit 1; }
TO=${GPU_TIMEOUT:-600}
exec timeout $((TO + 1500)) /usr/local/graft/bin/gpurun --timeout $TO -- "$@"
