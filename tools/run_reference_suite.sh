#!/usr/bin/env bash
# The reference package's own test suite (176 tests) with ircur.solve routed
# to the B200 drop-in (tools/ircur_dropin_plugin.py).
#
# Needs the reference installed in baseline/_ref and its
# tests copied next to it (baseline/_ref/reference_tests; git-ignored, travels
# to the GPU box with gpurun).  Writes gpurun_out/reference_suite.{log,xml}.
set -u
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
OUT="$ROOT/gpurun_out"
mkdir -p "$OUT" /tmp/dropin_run
cd /tmp/dropin_run
PYTHONPATH="$ROOT/tools:$ROOT" IRCUR_REF_SRC="$ROOT/baseline/_ref" \
  python -m pytest -p ircur_dropin_plugin -p no:cacheprovider -c /dev/null --rootdir=/tmp/dropin_run \
  "$ROOT/baseline/_ref/reference_tests" -q -rfE --junitxml="$OUT/reference_suite.xml" "$@" \
  > "$OUT/reference_suite.log" 2>&1
rc=$?
tail -40 "$OUT/reference_suite.log"
exit $rc
