#!/bin/bash
# time the tensor-core operator for each prebuilt library variant (tools/variants/*.so)
for lib in tools/variants/*.so; do
  for m in 0 3; do
    echo -n "$(basename $lib) "; NFS_B200_LIB=$lib NFS_TC_DEBUG=$m timeout 120 python tools/tc_modes.py 2>&1 | tail -1
  done
done
