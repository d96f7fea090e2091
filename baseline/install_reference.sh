#!/bin/sh
# Install the UNMODIFIED reference package (mdroute) into baseline/_ref for
# bench.py --impl reference.  Run once in the build container: /root/reference
# is read-only, so pip builds from a copy; numpy is already in the image, so
# dependency resolution is skipped (--no-deps).  baseline/_ref is git-ignored
# but travels to the GPU box with the repo snapshot.
set -e
cd "$(dirname "$0")/.."
rm -rf /tmp/mdroute_src && cp -r /root/reference/pkg /tmp/mdroute_src
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target baseline/_ref /tmp/mdroute_src
PYTHONPATH=baseline/_ref python -c "import mdroute; print('installed', mdroute.__file__)"
