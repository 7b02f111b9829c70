# build libmagnus_b200.so variants with -D knobs into variants/ (for on-box A/B sweeps)
set -e
cd "$(dirname "$0")/.."
build() {  # name, flags...
  local name=$1; shift
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
    --expt-relaxed-constexpr "$@" -o variants/lib_$name.so paper_2501_07056_b200/csrc/*.cu
}
build base &
build s6b0 -DMG_E2_BAL_SHORT=6 -DMG_E2_BAL_SEG=0 &
build s6b16 -DMG_E2_BAL_SHORT=6 -DMG_E2_BAL_SEG=16 &
build s8b16 -DMG_E2_BAL_SHORT=8 -DMG_E2_BAL_SEG=16 &
build s5b8 -DMG_E2_BAL_SHORT=5 -DMG_E2_BAL_SEG=8 &
wait
