#!/bin/bash
# Build an experiment variant of the whole library into
# paper_2509_10613_b200/_native/variants/<name>/libsigkernel.so (run it with
# SK_LIBSIGKERNEL=<that path>).  usage: tools/build_variant.sh <name> -DFLAG=...
set -e
cd "$(dirname "$0")/.."
python -m paper_2509_10613_b200.build --variant "$@"
