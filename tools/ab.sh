#!/bin/bash
# A/B timing of library variants on one box: tools/ab.sh <config> <lib1.so> <lib2.so> ... (two passes)
cfg=$1; shift
for pass in 1 2; do
  for lib in "$@"; do
    UBQP_LIB=$lib timeout 300 python tools/asc_sweep.py $cfg default 2>&1 | sed "s|^|$(basename $lib) |"
  done
done
