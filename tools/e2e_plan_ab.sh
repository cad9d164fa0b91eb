#!/bin/bash
# e2e chunk-plan A/B on config 1 (tools/e2e_trace.py): the last three call
# totals of gd_dock_batch per env setting.
CFGS=${CFGS:-"GD_E2E_CHUNKS=15|GD_E2E_GROWTH=1.5|GD_E2E_GROWTH=1.5 GD_E2E_HEAD=128|GD_E2E_GROWTH=1.5 GD_E2E_HEAD=128 GD_E2E_STREAMS=3|GD_E2E_GROWTH=1.75 GD_E2E_HEAD=128 GD_E2E_STREAMS=3|GD_E2E_GROWTH=1.5 GD_E2E_HEAD=64 GD_E2E_STREAMS=3|GD_E2E_GROWTH=2 GD_E2E_HEAD=64 GD_E2E_STREAMS=3|GD_E2E_GROWTH=1.5 GD_E2E_STREAMS=3"}
IFS='|' read -ra LIST <<< "$CFGS"
for cfg in "${LIST[@]}"; do
  echo "== $cfg"
  env $cfg GD_E2E_TRACE=1 timeout 300 python tools/e2e_trace.py 2>&1 | grep -E "call total" | tail -3 | tr '\n' ' '
  echo
done
