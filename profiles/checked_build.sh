# The checked library (device-side bounds / layout checks, -DCA_CHECKED) for
# tests/test_gpu_checked.py: built here into scratch/libs/checked.so (travels to the box).
set -e
cd "$(dirname "$0")/.."
python profiles/tune.py build checked=CA_CHECKED
