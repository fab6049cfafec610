#!/bin/bash
# AEG evict phase split (experiment build): pass c vs unit eviction
cd ${GRAFT_REPO_ROOT:-.}
VARIANTS="-DSAGA_TRACE_SPLIT4" bash scripts/gpu_ab2.sh
