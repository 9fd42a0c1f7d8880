#!/bin/bash
# Mixed-radix launch-shape sweep on the paper's 800x600 fp32 workload:
# gen_tune.sh "tcr:ntr:tcc:ntc ..." (empty field = the library's choice)
CFGS=${1:-"::: 1:64:1:64 2:64:2:64 1:32:1:32 2:128:2:128 4:128:4:128 8:256:8:256 1:128:1:128"}
for cfg in $CFGS; do
  IFS=: read -r tcr ntr tcc ntc <<< "$cfg"
  echo -n "TCR=$tcr NTR=$ntr TCC=$tcc NTC=$ntc: "
  PM_GEN_TCR=$tcr PM_GEN_NTR=$ntr PM_GEN_TCC=$tcc PM_GEN_NTC=$ntc timeout 120 python scripts/paper_config.py 2>&1 | tail -1 | sed 's/(incl.*download),//; s/; paper.*//'
done
