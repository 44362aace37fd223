#!/bin/bash
for lib in tools/variants/lib_seg*.so; do
  echo "== $lib"; NFS_B200_LIB=$lib PREC=f16x3 timeout 120 python tools/tc_modes.py; NFS_B200_LIB=$lib timeout 200 python tools/mask_diag.py | grep -E "q0|f16x3 res "
done
