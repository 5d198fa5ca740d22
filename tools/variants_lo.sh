#!/bin/bash
# kbench (all terms) at C3 degrees 1..3 (DEGS) for the default library and every build/variants/*.so
for so in default build/variants/*.so; do for p in ${DEGS:-1 2 3}; do
  if [ "$so" = default ]; then MASKS=all python tools/kbench.py C3 $p; else CUTFEM_LIB=$so MASKS=all python tools/kbench.py C3 $p; fi
done; done
