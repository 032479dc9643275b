#!/bin/bash
# Build the library here, then run a command on the B200 box (gpurun).
# Usage: tools/gpu.sh TIMEOUT_S 'command'
set -e
cd /root/repo
python -c "import __graft_entry__ as g; g.build()" > /tmp/gpu_build.log 2>&1 || { cat /tmp/gpu_build.log | tail -30; exit 1; }
/usr/local/graft/bin/gpurun --timeout "$1" -- "$2" > /tmp/gpurun_last.log 2>&1 || true
tail -3 /tmp/gpurun_last.log
