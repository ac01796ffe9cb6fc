#!/bin/bash
# K2 A/B across library builds: K2 ms at E in $ES for each build/lib_*.so named.
# Usage: scripts/k2_ab.sh TAG lib1 lib2 ...   (names of build/lib_<name>.so)
TAG=$1; shift
ES=${ES:-100,250,1000}
for name in "$@"; do
  echo "== $name"
  ARE_LIB=build/lib_$name.so timeout 300 python scripts/time_k2_e.py --es $ES 2>&1 | grep -v plan | tee gpurun_out/k2ab_${TAG}_$name.jsonl
done
