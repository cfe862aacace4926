#!/bin/bash
# p3s_convert per-call time under different environment settings (tools/pcie_probe.py).
for E in "$@"; do
  echo "$E: $(env $E timeout 120 python tools/pcie_probe.py 2>&1 | grep p3s_convert | tail -1)"
done
