#!/usr/bin/env bash
# compute-sanitizer passes over small invocations of every C-ABI entry point
# (memcheck, racecheck, synccheck, initcheck).  ONE tool per
# invocation (running several tools back to back in one process has left B200
# GPUs unusable on this driver, B200_PROFILING.md):  tests/sanitize.sh memcheck
set -euo pipefail
TOOL="${1:-memcheck}"
cd "$(dirname "$0")/.."
exec compute-sanitizer --tool "$TOOL" --error-exitcode 99 --print-limit 20 \
    python tools/sanitize_driver.py
