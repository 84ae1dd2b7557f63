#!/bin/bash
# libhhgstokes with device-side bounds checks (-DHHG_CHECKED) in every .cu -> paper_2506_04157_b200/lib/checked/
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
C=$ROOT/paper_2506_04157_b200/csrc; O=$ROOT/paper_2506_04157_b200/build/checked; mkdir -p $O $ROOT/paper_2506_04157_b200/lib/checked
PYSITE=$(python -c "import site;print([p for p in site.getsitepackages() if 'site-packages' in p][0])")
NCCL=$PYSITE/nvidia/nccl
ARCH="-gencode arch=compute_100a,code=sm_100a"
for f in hhg_mesh hhg_elem hhg_kernels hhg_capi hhg_mg hhg_comm hhg_temp; do
  nvcc $ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 -I$NCCL/include --expt-relaxed-constexpr -DHHG_CHECKED -c $C/$f.cu -o $O/$f.o &
done
wait
nvcc $ARCH -shared -o $ROOT/paper_2506_04157_b200/lib/checked/libhhgstokes.so $O/*.o -L$NCCL/lib -l:libnccl.so.2 -Xlinker -rpath,$NCCL/lib -lcudart
echo built checked/libhhgstokes.so
