#!/bin/bash
# Build the committed HEAD's libotg.so into ab/head/ (reference arm of A/B runs)
set -e
cd "$(dirname "$0")/.."
rm -rf /tmp/abhead && mkdir -p /tmp/abhead && git archive HEAD paper_2605_30267_b200 include | tar -x -C /tmp/abhead
(cd /tmp/abhead && python -c "import sys; sys.path.insert(0,'.'); from paper_2605_30267_b200 import build as B; B.build()" > /dev/null)
mkdir -p ab/head && cp /tmp/abhead/paper_2605_30267_b200/libotg.so ab/head/libotg.so && echo "built ab/head/libotg.so ($(git rev-parse --short HEAD))"
