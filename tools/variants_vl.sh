for so in default build/variants/*.so; do for p in 4 5 6 7 8; do
  if [ "$so" = default ]; then MASKS=all python tools/kbench.py C3 $p; CUTFEM_NO_VLINES=1 MASKS=all python tools/kbench.py C3 $p | sed 's/"default"/"novlines"/'; else CUTFEM_LIB=$so MASKS=all python tools/kbench.py C3 $p; fi
done; done
MASKS=all python tools/kbench.py C5; CUTFEM_NO_VLINES=1 MASKS=all python tools/kbench.py C5 | sed 's/"default"/"novlines"/'
