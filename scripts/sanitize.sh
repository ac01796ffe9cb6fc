#!/bin/bash
# compute-sanitizer over the edge-case parity tests (run on the GPU box).
set -o pipefail
K='worked or empty_trial or nan_inf or 256_tables or long_and_ragged or slot_zero or out_of_range or degenerate or large_catalogs'
compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -x -q -k "$K" 2>&1 | tail -3
L='dense_overlap_and_odd_layer_counts and (5 or 7)'
compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -x -q -k "$L" 2>&1 | tail -3
compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -x -q -k "long_and_ragged or 256_tables" 2>&1 | tail -3
compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -x -q -k "$L" 2>&1 | tail -3
compute-sanitizer --tool synccheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -x -q -k "long_and_ragged or 256_tables" 2>&1 | tail -3
# the cooperative event-major dense kernel (k2_dense_coop, one- and two-line strides, FULL and generic shapes)
D='dense_overlap_plans_event_major_kernel'
compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -x -q -k "$D" 2>&1 | tail -3
compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -x -q -k "$D" 2>&1 | tail -3
compute-sanitizer --tool synccheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -x -q -k "$D" 2>&1 | tail -3
