#!/bin/bash
# build a variant of the library with extra nvcc flags for nfs_tci.cu:  tools/build_variant.sh NAME -DFOO=1 ...
# (TCI_SRC=path compiles another copy of nfs_tci.cu, e.g. `git show HEAD:...` for A/B runs)
set -e
cd "$(dirname "$0")/.."
python -m paper_2604_09233_b200.build >/dev/null
name=$1; shift
mkdir -p tools/variants build/variants
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-fopenmp -Xptxas -O3 -Iinclude "$@" \
  -Ipaper_2604_09233_b200/csrc -c ${TCI_SRC:-paper_2604_09233_b200/csrc/nfs_tci.cu} -o build/variants/nfs_tci_$name.o
objs=$(ls build/nfs_b200/*.o | grep -v nfs_tci.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o tools/variants/lib_$name.so $objs build/variants/nfs_tci_$name.o -ldl -lgomp
echo tools/variants/lib_$name.so
