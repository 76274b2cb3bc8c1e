#!/usr/bin/env bash
# Build the C++ façade test program against the in-tree library (called by __graft_entry__.build()).
set -euo pipefail
ROOT="$(cd "$(dirname "${BASH_SOURCE[0]}")/../.." && pwd)"
g++ -std=c++17 -O2 -Wall -Wextra -I "$ROOT/include" "$ROOT/tests/cpp/test_facade.cpp" \
    -L "$ROOT/paper_2507_02809_b200" -l:libfracinv_b200.so -Wl,-rpath,'$ORIGIN/../../paper_2507_02809_b200' \
    -o "$ROOT/tests/cpp/test_facade"
