#!/bin/bash
for cfg in "16 4 2" "16 4 3" "16 4 4" "16 2 4" "16 8 3" "32 4 3" "16 4 2"; do
  set -- $cfg
  echo "T=$1 MB=$2 NB=$3"; CAFS_XFER_T=$1 CAFS_XFER_MB=$2 CAFS_XFER_NB=$3 timeout 300 python scratch/pageable_e2e.py 2>&1 | grep "2^30"
done
