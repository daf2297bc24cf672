#!/bin/bash
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
echo "--- PDL on"; bash scratch/quick_bench.sh cfg1 cfg2 cfg3 cfg4 cfg5
echo "--- PDL off"; CAFS_PDL=0 bash scratch/quick_bench.sh cfg1 cfg2 cfg4
