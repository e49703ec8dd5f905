#!/bin/sh
# Build an A/B variant of libwm3.so with extra nvcc defines into tools/_variants/<name>/libwm3.so (git-ignored);
# select it at run time with WM3_LIB=tools/_variants/<name>/libwm3.so.
#   tools/build_variant.sh emu2 -DWM3_NA_EMU=2
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
NAME=$1; shift
OUT=$ROOT/tools/_variants/$NAME
mkdir -p "$OUT"
make -C "$ROOT" -s clean >/dev/null 2>&1 || true
rm -rf "$ROOT/build"
make -C "$ROOT" -s -j16 NVFLAGS_EXTRA="$*" >/dev/null
cp "$ROOT/paper_2503_22235_b200/libwm3.so" "$OUT/libwm3.so"
echo "$OUT/libwm3.so"
# restore the default build
rm -rf "$ROOT/build"
make -C "$ROOT" -s -j16 >/dev/null
