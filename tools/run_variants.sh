#!/bin/bash
# Time quick_time's "k1" set under each variants/lib_*.so (development A/B aid).
for lib in variants/lib_*.so; do
  echo "== $lib"
  PFT_LIB=$lib QT=${QT:-k1} python tools/quick_time.py 2>&1 | grep -v Warning
done
