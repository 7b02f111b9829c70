# build libmagnus_b200.so variants with -D knobs into variants/ (for on-box A/B sweeps)
# usage: tools/build_variants.sh name "-DFLAG=.. -DFLAG2=.." [name "flags"] ...
set -e
cd "$(dirname "$0")/.."
mkdir -p variants
while [ $# -gt 1 ]; do
  name=$1; flags=$2; shift 2
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
    --expt-relaxed-constexpr $flags -o variants/lib_$name.so paper_2501_07056_b200/csrc/*.cu &
done
wait
