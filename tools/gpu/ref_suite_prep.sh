# build container only: copy the reference's tests next to its pip install (both git-ignored, both travel)
cd "$(dirname "$0")/../.."
rm -rf baseline/_ref_tests && cp -r /root/reference/pkg/tests baseline/_ref_tests
