# build a libsonic variant to exp_libs/<name>.so: bash tools/build_variant.sh name "-DFLAG=.."
set -e
cd "$(dirname "$0")/../paper_2512_14080_b200"
mkdir -p ../exp_libs
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC \
  -Xcompiler -O3 $2 -o ../exp_libs/$1.so csrc/sonic_api.cu csrc/route.cu csrc/aggregate.cu csrc/ep.cu csrc/peer.cu csrc/router.cu csrc/fp8.cu
