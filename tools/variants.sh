#!/bin/bash
# run kbench for the default library and every build/variants/*.so (one GPU call)
CFG=${1:-C2}
for so in default build/variants/*.so; do
  if [ "$so" = default ]; then MASKS=${MASKS:-all,cell,none} python tools/kbench.py $CFG; else CUTFEM_LIB=$so MASKS=${MASKS:-all,cell,none} python tools/kbench.py $CFG; fi
done
