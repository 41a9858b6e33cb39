#!/bin/bash
# permute grid cap sweep: permute alone, and concurrent with the schedule build
for g in 1 2 3 4 6 8; do
  echo "SCFA_PERM_G=$g"
  SCFA_PERM_G=$g python scripts/scratch/permute_prio.py 2>&1 | grep -v range
done
