#!/usr/bin/env bash
# Regenerates tests/golden/ref_infra.json from the reference's own shipped rng.hpp /
# parallel.hpp / binary_io.cpp (compiled by `make -C oracle ref`). TEST INFRASTRUCTURE ONLY.
set -euo pipefail
here="$(cd "$(dirname "$0")" && pwd)"
make -C "$here" ref >/dev/null
"$here/_ref/ref_golden" "$(mktemp)" > "$here/../tests/golden/ref_infra.json"
echo "wrote tests/golden/ref_infra.json"
