#!/usr/bin/env bash
# Experiment helper: build libsnop_cuda.so with extra nvcc flags into tmp_exp/<name>.so
# (separate object directory; the in-tree build is untouched). Usage: build_variant.sh name "-DFOO=1 ..."
set -euo pipefail
name="$1"; extra="${2:-}"
root="$(cd "$(dirname "$0")/.." && pwd)"
work="/tmp/snop_variant_$name"
rm -rf "$work"; mkdir -p "$work/paper_2509_01416_b200" "$root/tmp_exp"
cp -r "$root/paper_2509_01416_b200/csrc" "$work/paper_2509_01416_b200/"
cp -r "$root/include" "$work/"
rm -f "$work"/paper_2509_01416_b200/csrc/*.o
make -C "$work/paper_2509_01416_b200/csrc" -j8 NVFLAGS="-O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr $extra" OUT="$root/tmp_exp/$name.so" >/dev/null
grep -h "spill" "$work"/paper_2509_01416_b200/csrc/si_k8_fixed.o.ptxas.log | sort | uniq -c | sort -rn | head -3 || true
echo "built tmp_exp/$name.so"
