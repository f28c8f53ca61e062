# The reference's own test suite (baseline/_ref_tests = copy of /root/reference/pkg/tests, made in the build
# container by tools/gpu/ref_suite_prep.sh) with the B200 kernels as its backend (tools/ref_suite_b200.py).
cd "$(dirname "$0")/../.."
cd baseline/_ref_tests && PYTHONPATH=../..:../_ref:../../tools python -m pytest -q -p ref_suite_b200 . "$@"
