#!/bin/bash
# build_variant.sh NAME "FLAGS" : libhhgstokes variant with hhg_elem.cu compiled with extra -D flags
# -> paper_2506_04157_b200/lib/exp_NAME.so (A/B timing via HHG_LIB; never the product path)
set -e
NAME=$1; FLAGS=$2
ROOT=$(cd "$(dirname "$0")/.." && pwd)
C=$ROOT/paper_2506_04157_b200/csrc; B=$ROOT/paper_2506_04157_b200/build; O=$B/exp_$NAME; mkdir -p $O
PYSITE=$(python -c "import site;print([p for p in site.getsitepackages() if 'site-packages' in p][0])")
NCCL=$PYSITE/nvidia/nccl
ARCH="-gencode arch=compute_100a,code=sm_100a"
make -s -C $C >/dev/null
nvcc $ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 -I$NCCL/include --expt-relaxed-constexpr $FLAGS -c $C/hhg_elem.cu -o $O/hhg_elem.o
OBJS=$(ls $B/*.o | grep -v hhg_elem.o)
nvcc $ARCH -shared -o $ROOT/paper_2506_04157_b200/lib/exp_$NAME.so $O/hhg_elem.o $OBJS -L$NCCL/lib -l:libnccl.so.2 -Xlinker -rpath,$NCCL/lib -lcudart
echo built exp_$NAME.so
