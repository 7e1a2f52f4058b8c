# The unmodified reference for the bench's reference arm and the replay of its
# own test-suite through the drop-in (tests/test_gpu_reference_suite.py):
# pip-installs /root/reference/pkg (from a copy: the tree is read-only) into
# baseline/_ref (git-ignored, shipped to the GPU box by gpurun) and copies the
# reference's pkg/tests next to it as baseline/_ref/reference_tests.
# numpy / numba / click come from the image (--no-deps).
set -e
cd "$(dirname "$0")/.."
rm -rf /tmp/evd_refcopy baseline/_ref
cp -r /root/reference /tmp/evd_refcopy
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target baseline/_ref /tmp/evd_refcopy/pkg
mkdir -p baseline/_ref/reference_tests
cp /root/reference/pkg/tests/*.py baseline/_ref/reference_tests/
rm -rf /tmp/evd_refcopy
echo "installed: $(ls baseline/_ref)"
