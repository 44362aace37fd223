#!/bin/bash
# Stage the UNMODIFIED reference package (build container only; /root/reference does not exist
# on the GPU box).  Both directories are git-ignored but travel to the box with the snapshot:
#   baseline/_ref        pip install of /root/reference/pkg (--no-deps: matplotlib is absent and
#                        only the report figures need it); the reference arm of bench.py and the
#                        drop-in checks import `nfsense` from here
#   baseline/_ref_tests  the reference's own test files (pkg/tests), run unchanged through the
#                        GPU dispatch by tests/test_gpu_reference_suite.py
set -e
cd "$(dirname "$0")/.."
src=/root/reference/pkg
tmp=$(mktemp -d)
cp -r "$src" "$tmp/pkg"          # the setuptools build writes into its source tree
rm -rf baseline/_ref baseline/_ref_tests
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
  --target baseline/_ref "$tmp/pkg" >/dev/null
cp -r "$src/tests" baseline/_ref_tests
rm -rf "$tmp"
echo "staged baseline/_ref ($(ls baseline/_ref)) and baseline/_ref_tests"
