#!/usr/bin/env bash
# Builds libfgfrft_b200.so in-tree for sm_100a (called by __graft_entry__.build()).
set -euo pipefail
HERE="$(cd "$(dirname "${BASH_SOURCE[0]}")" && pwd)"
ROOT="$(dirname "$HERE")"
NVCC="${NVCC:-/usr/local/cuda/bin/nvcc}"
OUT="$HERE/libfgfrft_b200.so"
SRC="$HERE/csrc"
OBJ="$HERE/build"
mkdir -p "$OBJ"
FLAGS=(-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC
       -Xcompiler -ffp-contract=off -I"$ROOT/include" -I"$SRC" --expt-relaxed-constexpr)
[ -n "${FGFRFT_PTXAS_VERBOSE:-}" ] && FLAGS+=(-Xptxas -v)
pids=()
for f in capi capi_shard capi_learn capi_spectral capi_store synth zgemm cgemm dots ops layout shard batch real ozgemm combine denoise spectral store packed capi_pshard; do
  "$NVCC" "${FLAGS[@]}" -c "$SRC/$f.cu" -o "$OBJ/$f.o" & pids+=($!)
done
"$NVCC" "${FLAGS[@]}" -x cu -c "$SRC/sinc_host.cpp" -o "$OBJ/sinc_host.o" & pids+=($!)
for p in "${pids[@]}"; do wait "$p"; done
"$NVCC" -gencode arch=compute_100a,code=sm_100a -shared -o "$OUT" "$OBJ"/*.o -lcudart -ldl
echo "built $OUT"
