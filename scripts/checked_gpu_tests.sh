#!/bin/bash
# Run the GPU suite against the checked build (device bounds assertions, ADAKV_DCHECK), then
# restore the shipped build.  Usage (on a GPU box): scripts/checked_gpu_tests.sh
set -u
cd "$(dirname "$0")/.."
make -s -C paper_2407_11550_b200/csrc clean >/dev/null
make -s -j16 -C paper_2407_11550_b200/csrc EXTRA=-DADAKV_DEVICE_CHECKS || exit 1
python -m pytest tests -m gpu -q -p no:cacheprovider
rc=$?
make -s -C paper_2407_11550_b200/csrc clean >/dev/null
make -s -j16 -C paper_2407_11550_b200/csrc
exit $rc
