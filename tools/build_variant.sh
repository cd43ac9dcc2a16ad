# Build an A/B variant of the library with extra nvcc defines into paper_2506_20252_b200/libpatb200_<name>.so
# (loaded when PAT_LIB_VARIANT=<name>):  bash tools/build_variant.sh poll16 -DPAT_LL32_POLL16=1
set -e
NAME=$1; shift
R=$(cd "$(dirname "$0")/.." && pwd)
make -s -j8 -C $R/paper_2506_20252_b200/csrc OBJ=$R/paper_2506_20252_b200/csrc/build_$NAME \
  OUT=$R/paper_2506_20252_b200/libpatb200_$NAME.so NVCC="/usr/local/cuda/bin/nvcc $*"
