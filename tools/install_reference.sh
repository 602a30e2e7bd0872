#!/bin/bash
# Installs the unmodified reference (ringmix) into baseline/_ref (git-ignored; travels to the
# GPU box with the gpurun snapshot) plus a copy of its own test files under
# baseline/_ref/ringmix_ref_tests, which tests/test_gpu_reference_suite.py runs through the
# libringmix_b200 binding (integration/ringmix_b200.py).  Offline: the image's wheelhouse.
set -e
cd "$(dirname "$0")/.."
[ -d /root/reference/pkg ] || { echo "no /root/reference here"; exit 0; }
rm -rf /tmp/ringmix_src && cp -r /root/reference/pkg /tmp/ringmix_src
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
  --target baseline/_ref /tmp/ringmix_src > baseline_install.log 2>&1 || { cat baseline_install.log; exit 1; }
rm -rf baseline/_ref/ringmix_ref_tests && cp -r /root/reference/pkg/tests baseline/_ref/ringmix_ref_tests
rm -f baseline_install.log
echo "installed: $(ls baseline/_ref)"
