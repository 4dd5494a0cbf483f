#!/bin/bash
# Install the UNMODIFIED reference package (mxcomm, pure Python + numpy) into
# baseline/_ref -- git-ignored, but shipped to the GPU box by gpurun -- for
# bench.py's reference arm and cpu_baseline.  The build writes into its
# source tree, so it runs from a copy under /tmp (/root/reference is
# read-only).  Offline: no index, no dependency resolution (numpy is in the
# image).
set -euo pipefail
cd "$(dirname "$0")/.."
rm -rf /tmp/mxcomm_ref_src baseline/_ref
cp -r /root/reference/pkg /tmp/mxcomm_ref_src
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
  --target baseline/_ref /tmp/mxcomm_ref_src
PYTHONPATH=baseline/_ref python -c "import mxcomm, sys; print('installed', mxcomm.__file__)"
