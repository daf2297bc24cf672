#!/bin/bash
for m in 0xff 0 0xf7 0xef 0xf3 0x7f 0xfb; do echo "mask $m"; CAFS_PDL=$m bash scratch/quick_bench.sh cfg3; done
