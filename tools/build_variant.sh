#!/bin/bash
# build a variant of the library with extra nvcc flags for one source (default nfs_tci.cu):
#   tools/build_variant.sh NAME -DFOO=1 ...          (VAR_SRC=nfs_tc picks csrc/nfs_tc.cu)
# (TCI_SRC=path compiles another copy of the source, e.g. `git show HEAD:...` for A/B runs)
set -e
cd "$(dirname "$0")/.."
python -m paper_2604_09233_b200.build >/dev/null
name=$1; shift
src=${VAR_SRC:-nfs_tci}
mkdir -p tools/variants build/variants
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-fopenmp -Xptxas -O3 -Iinclude "$@" \
  -Ipaper_2604_09233_b200/csrc -c ${TCI_SRC:-paper_2604_09233_b200/csrc/$src.cu} -o build/variants/${src}_$name.o
objs=$(ls build/nfs_b200/*.o | grep -v "/$src.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o tools/variants/lib_$name.so $objs build/variants/${src}_$name.o -ldl -lgomp
echo tools/variants/lib_$name.so
