#!/bin/bash
# Install the UNMODIFIED reference package (pnce) into baseline/_ref (git-ignored, travels to
# the GPU box with gpurun) so the GPU tests can run the INTEGRATION.md binding on the
# reference's own objects.  /root/reference is read-only: build from a copy under /tmp.
set -e
cd "$(dirname "$0")/.."
rm -rf /tmp/pnce_ref_src baseline/_ref
cp -r /root/reference/pkg /tmp/pnce_ref_src
python -m pip install --no-index --no-build-isolation --find-links /opt/wheelhouse \
    --target baseline/_ref /tmp/pnce_ref_src --no-deps
python -c "import sys; sys.path.insert(0, 'baseline/_ref'); import pnce.experiments; print('pnce installed:', pnce.__file__)"
