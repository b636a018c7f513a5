#!/bin/sh
# Rebuild libcotten.so only (the package import would load the stale library).
cd "$(dirname "$0")/.." && python -c "import __graft_entry__ as g; g._build_module().build_cuda(force=True)"
