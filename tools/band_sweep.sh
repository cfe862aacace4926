for E in "" "1,4,8,12,14,16" "1,3,6,9,12,14,16" "1,5,9,13,15,16" "2,6,10,14,16"; do
  echo "ends=$E"; if [ -z "$E" ]; then unset P3S_BAND_ENDS; else export P3S_BAND_ENDS=$E; fi; P3S_DEBUG_CONV=1 timeout 120 python tools/pcie_probe.py 2>&1 | tail -3
done
