#!/usr/bin/env bash
# Compile the REFERENCE's own unit tests and acceptance gate, unmodified, from
# /root/reference/proj/tests against this repo's drop-in headers
# (include/qzsim) and libqzsim_b200.so, with tests/cpp/doctest.h standing in
# for the absent doctest.  Binaries go to build/reftests/ (not committed;
# they travel to the GPU box as built artefacts, like the .so files).
# test_qasm is skipped: the QASM parser is out of scope.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/../.." && pwd)"
REF="${REF:-/root/reference/proj/tests}"
JSON_DIR="${JSON_DIR:-/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann}"
OUT="$ROOT/build/reftests"
LIB="$ROOT/paper_2309_16979_b200/lib"
[ -d "$REF" ] || { echo "no reference tests at $REF"; exit 0; }
mkdir -p "$OUT"
for t in test_codec test_store test_planner test_device test_pipeline test_gates test_oracle acceptance; do
  g++ -std=gnu++20 -O2 -I"$ROOT/include" -I"$ROOT/tests/cpp" -I"$JSON_DIR" \
      "$REF/$t.cpp" -o "$OUT/$t" -L"$LIB" -lqzsim_b200 -lqzcuda -Wl,-rpath,"$LIB" &
done
wait
ls "$OUT"
