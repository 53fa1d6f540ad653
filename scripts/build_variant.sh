# build an A/B variant of libgpcg.so into build_variants/NAME.so with extra nvcc flags
# usage: bash scripts/build_variant.sh NAME "-DGPCG_GP_SPEC6=0 ..."   (select it with GPCG_LIB=build_variants/NAME.so)
set -e
mkdir -p build_variants
/usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo --extended-lambda \
  -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -shared -I include -I paper_cs_0101018_b200/csrc -ldl $2 \
  -o build_variants/$1.so paper_cs_0101018_b200/csrc/gpcg.cu
