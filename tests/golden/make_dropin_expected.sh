#!/bin/sh
# Regenerates tests/golden/dropin_expected.txt: tests/cpp/dropin_scenarios.cpp
# compiled against the UNMODIFIED reference headers (needs /root/reference,
# i.e. the dev container) and run on the CPU.
set -e
HERE=$(cd "$(dirname "$0")" && pwd)
make -C "$HERE/../../oracle" dropin
"$HERE/../../oracle/_ref/dropin_scenarios_ref" > "$HERE/dropin_expected.txt"
