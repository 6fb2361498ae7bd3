#!/usr/bin/env bash
# Device-side invariant checks instead of compute-sanitizer (closed on this
# GPU pool): builds libphmat_b200_checked.so (PHM_DCHECK traps on the layout
# assumptions of the TMA / shared-memory kernels) and runs the small
# all-kernels workload of tools/sanitize_run.py plus the GPU parity tests on
# it. Run from the repo root on a B200.
set -eu
make -C paper_2511_03109_b200 checked > /dev/null
PHM_LIB=libphmat_b200_checked.so python tools/sanitize_run.py
PHM_LIB=libphmat_b200_checked.so python -m pytest tests -m gpu -x -q 2>&1 | tail -2
