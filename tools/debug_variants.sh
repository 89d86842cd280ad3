#!/bin/bash
# run the stage check under several library variants (development aid)
for lib in paper_2008_12559_b200/libpft_b200.so variants/lib_PFT_DBG_SYNCWARP.so variants/lib_PFT_DBG_STAGES2.so variants/lib_PFT_DBG_ONE_CTA.so variants/lib_PFT_DBG_BULK1D.so; do
  echo "== $lib"
  PFT_LIB=$lib python - <<'PY'
import sys; sys.path.insert(0, "tools"); sys.path.insert(0, ".")
import debug_stages as d
for rep in range(2):
    d.check(2**24, 2**10, 2**22, 2**15); print("  bad residues:", d.LAST)
d.check(2**24, 2**10, 2**22, 2**16)
PY
done
