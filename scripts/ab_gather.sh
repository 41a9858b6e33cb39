#!/bin/bash
# A/B of the bucket-order copy kernels across builds in ab/ (diagnostics)
for lib in ab/*.so; do echo "== $lib"; SCFA_LIB=$GRAFT_REPO_ROOT/$lib timeout 120 python scripts/gather_timing.py 2>&1 | head -2; done
