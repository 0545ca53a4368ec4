#!/bin/bash
# Golden output of the reference's acceptance suite (proj/tests/acceptance.cpp) compiled AS-IS
# against the reference headers on the CPU: tests/golden/reference_acceptance.txt.  The GPU test
# tests/test_cpp_dropin.py::test_reference_acceptance_suite_against_dropin compares the same suite
# compiled against the B200 drop-in header with it, criterion by criterion.
set -e
REF=${REF:-/root/reference/proj}
ROOT=$(cd "$(dirname "$0")/.." && pwd)
g++ -std=c++20 -O2 -I"$REF/include" -I"$REF/tests" "$REF/tests/acceptance.cpp" -o /tmp/tcr_acceptance_ref
/tmp/tcr_acceptance_ref > "$ROOT/tests/golden/reference_acceptance.txt" || true
cat "$ROOT/tests/golden/reference_acceptance.txt"
