#!/bin/bash
# Mixed-radix plan sweep (radix cap, pass order, launch shape) on the paper's 800x600 fp32 workload.
for o in ${ORDERS:-0 1 2}; do for r in ${RMAXS:-8 12 16 32}; do for cfg in ${CFGS:-1:256:2:256 2:128:2:128 8:256:8:256}; do
  IFS=: read -r tcr ntr tcc ntc <<< "$cfg"
  echo -n "ORDER=$o RMAX=$r TCR=$tcr NTR=$ntr TCC=$tcc NTC=$ntc: "
  PM_GEN_ORDER=$o PM_GEN_RMAX=$r PM_GEN_TCR=$tcr PM_GEN_NTR=$ntr PM_GEN_TCC=$tcc PM_GEN_NTC=$ntc timeout 120 python scripts/paper_config.py 2>&1 | tail -1 | sed 's/(incl.*download),//; s/; paper.*//; s/800x600 fp32, 25 GS iterations://'
done; done; done
