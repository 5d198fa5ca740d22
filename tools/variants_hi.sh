#!/bin/bash
# kbench (all terms) at C3 degrees 4..8 for the default library and every build/variants/*.so
for so in default build/variants/*.so; do
  for p in ${DEGS:-4 5 6 7 8}; do
    if [ "$so" = default ]; then MASKS=all python tools/kbench.py C3 $p; else CUTFEM_LIB=$so MASKS=all python tools/kbench.py C3 $p; fi
  done
done
