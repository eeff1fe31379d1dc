#!/bin/bash
# The checked build (device-side SKH_CHECK invariants, csrc/common.cuh) under the
# whole GPU suite -- the stand-in for compute-sanitizer, closed on the GPU pool.
# SKH_CHECKED stays exported so the tests' build() calls keep the checked library.
export SKH_CHECKED=1
python -m paper_2105_11815_b200.build || exit 1
python -m pytest tests -m gpu -q "$@"
rc=$?
unset SKH_CHECKED
python -m paper_2105_11815_b200.build > /dev/null   # back to the product build
exit $rc
