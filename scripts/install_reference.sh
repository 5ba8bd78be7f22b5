#!/bin/sh
# Offline install of the unmodified reference package into baseline/_ref
# (git-ignored, shipped to the GPU box by gpurun), plus its own test modules
# under baseline/_ref/tests for tests/test_reference_dropin.py, which runs
# them against this backend.  Nothing here is committed.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
rm -rf /tmp/gf_ref_src && cp -r /root/reference/pkg /tmp/gf_ref_src
python -m pip install --no-index --no-build-isolation --find-links /opt/wheelhouse --target "$ROOT/baseline/_ref" /tmp/gf_ref_src
mkdir -p "$ROOT/baseline/_ref/tests"
cp /root/reference/pkg/tests/test_interpreter.py /root/reference/pkg/tests/_graphgen.py "$ROOT/baseline/_ref/tests/"
