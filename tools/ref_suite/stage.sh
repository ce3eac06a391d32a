#!/bin/sh
# Stage the reference's own tests (read-only upstream, not committed: baseline/ is
# git-ignored) next to its offline install so run_ref_suite.py can run them on the GPU box.
set -e
ROOT=$(cd "$(dirname "$0")/../.." && pwd)
mkdir -p "$ROOT/baseline/_ref_tests"
cp /root/reference/pkg/tests/*.py "$ROOT/baseline/_ref_tests/"
if [ ! -d "$ROOT/baseline/_ref/gooms" ]; then
  rm -rf /tmp/_gooms_pkg && cp -r /root/reference/pkg /tmp/_gooms_pkg
  python -m pip install --no-index --no-build-isolation --no-deps --target "$ROOT/baseline/_ref" /tmp/_gooms_pkg
fi
ls "$ROOT/baseline/_ref_tests"
