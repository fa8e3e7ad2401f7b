#!/bin/bash
# r02b: conv_run_host with the planned chunks vs equal-chunk alternatives
cd "$(dirname "$0")/.."
for path in fp32_simt fp32_tc bf16 tf32; do
  for c in "" 4 6 8 16; do
    for rep in 1 2; do echo "$path ${c:-plan} $(CONV_HOST_CHUNKS=$c python scripts/probe_e2e.py --one $path batched)"; done
  done
done
