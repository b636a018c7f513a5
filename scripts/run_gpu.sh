#!/bin/bash
# Build everything in-tree (the .so files travel with the snapshot), then run
# the given script on a B200 through gpurun.
set -e
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" > /tmp/build.log 2>&1 || { tail -20 /tmp/build.log; exit 1; }
/usr/local/graft/bin/gpurun --timeout "${GPU_TIMEOUT:-1800}" -- "bash $1"
