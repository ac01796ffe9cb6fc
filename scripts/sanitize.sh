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
# round 2: the relay kernel (k2_relay: TMA filter load, mbarrier ring between producer and fold warps,
# texture gathers, NaN-tagged records) and the multi-GPU group (per-shard uploads, peer gather).
# synccheck/racecheck track every mbarrier (148 CTAs x 129): raise their table or they overflow.
R='ragged_trials_across_the_stream or short_trials_in_the_relay_range or occurrence_terms_sweep'
compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_relay.py -x -q -k "$R" 2>&1 | tail -3
compute-sanitizer --tool memcheck --error-exitcode 9 python scripts/relay_small.py 2>&1 | tail -2
compute-sanitizer --tool synccheck --num-cuda-barriers 40000 --error-exitcode 9 python scripts/relay_small.py 2>&1 | tail -2
compute-sanitizer --tool racecheck --num-cuda-barriers 40000 --print-limit 4 python scripts/relay_small.py 2>&1 | tail -6
compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_group.py tests/test_gpu_concurrency.py -x -q 2>&1 | tail -3
# round 2, late: the packed-id stream of the relay kernel (k2_relay<..., PK=true>) and the packing kernel
compute-sanitizer --tool memcheck --error-exitcode 9 python scripts/relay_small.py --packed 2>&1 | tail -2
compute-sanitizer --tool synccheck --num-cuda-barriers 40000 --error-exitcode 9 python scripts/relay_small.py --packed 2>&1 | tail -2
compute-sanitizer --tool racecheck --num-cuda-barriers 40000 --print-limit 4 python scripts/relay_small.py --packed 2>&1 | tail -6
compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_packed.py -x -q -k "layout or subrange or wide" 2>&1 | tail -3
