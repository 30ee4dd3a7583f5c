#!/bin/bash
# A/B timing of library variants on one box (two passes):
#   tools/ab.sh <config|micro> <lib1.so> <lib2.so> ...
cfg=$1; shift
for pass in 1 2; do
  for lib in "$@"; do
    if [ "$cfg" = micro ]; then UBQP_LIB=$lib timeout 300 python tools/asc_micro.py 2>&1 | sed "s|^|$(basename $lib) |"; else UBQP_LIB=$lib timeout 300 python tools/asc_sweep.py $cfg default 2>&1 | sed "s|^|$(basename $lib) |"; fi
  done
done
