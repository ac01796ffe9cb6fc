#!/bin/bash
# K2 A/B across build/lib_<name>.so builds, then one ncu --set full capture of
# the first build's relay/hot-set kernel.  Usage: scripts/ab_ncu.sh TAG lib1 lib2 ...
TAG=$1; shift
ES=${ES:-500,1000,2000} bash scripts/k2_ab.sh $TAG "$@"
ARE_LIB=build/lib_$1.so ncu --set full --clock-control none --import-source on -k regex:"k2_(relay|hotset)" -s 1 -c 1 \
    -o gpurun_out/k2_$TAG python scripts/profile_k2.py --launches 2 > gpurun_out/ncu_$TAG.log 2>&1
tail -1 gpurun_out/ncu_$TAG.log
