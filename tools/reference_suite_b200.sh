# The reference's own test suite against the B200 backend (integration/):
# install the binding into a copy of the built reference, run every test
# file with ILANS_BACKEND=b200, then the derived TestKernelEquivalence.
set -u
dest=/tmp/ilans_ref_b200
python integration/install_into_reference.py $dest > /dev/null
lib=$(python -c "from paper_1402_3392_b200 import _lib; print(_lib.LIB_PATH)")
cd $dest
ILANS_BACKEND=b200 ILANS_B200_LIB=$lib PYTHONPATH=$dest python -m pytest tests -q -p no:cacheprovider \
    --deselect tests/test_backend.py::TestSelection::test_ext_resolves -rs 2>&1 | tail -8
echo "---- derived: TestKernelEquivalence, pure vs b200"
ILANS_BACKEND=b200 ILANS_B200_LIB=$lib PYTHONPATH=$dest python -m pytest tests/test_backend_b200.py -v \
    -p no:cacheprovider -k TestKernelEquivalence 2>&1 | grep -E "PASSED|FAILED|passed|failed"
