#!/bin/bash
# Mixed-radix launch-shape sweep on the paper's 800x600 fp32 workload.
for tcr in 1 2 4; do for tcc in 2 4; do for nt in 128 256 384; do
  echo -n "TCR=$tcr TCC=$tcc NT=$nt: "
  PM_GEN_TCR=$tcr PM_GEN_TCC=$tcc PM_GEN_NTR=$nt PM_GEN_NTC=$nt timeout 120 python scripts/paper_config.py 2>&1 | tail -1 | sed 's/(incl.*download),//; s/; paper.*//'
done; done; done
