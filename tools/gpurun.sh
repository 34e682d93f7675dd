#!/bin/bash
# Rebuild every in-tree library here, then run a command on the B200 box:
# the snapshot ships the built .so files, so a stale build would be measured.
# Usage: tools/gpurun.sh TIMEOUT_S 'command'
set -e
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" > build/last_build.log 2>&1 || { tail -30 build/last_build.log; exit 1; }
exec /usr/local/graft/bin/gpurun --timeout "$1" -- "$2"
