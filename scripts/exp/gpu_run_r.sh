#!/bin/bash
# BELADY evict phase split: threshold searches (slot 2) / take-all-dead (slot 3) / the rest (slot 4)
cd ${GRAFT_REPO_ROOT:-.}
VARIANTS="" bash scripts/gpu_ab2.sh
