#!/bin/bash
# kbench of one config/degree for the default library and every build/variants/*.so
CFG=${1:-C3}; DEG=${2:-4}
for so in default build/variants/*.so; do
  if [ "$so" = default ]; then MASKS=${MASKS:-all} python tools/kbench.py $CFG $DEG; else CUTFEM_LIB=$so MASKS=${MASKS:-all} python tools/kbench.py $CFG $DEG; fi
done
