#!/bin/bash
# compute-sanitizer over the GPU parity tests (run under gpurun).  Each tool runs a
# subset of tests/test_gpu_parity.py chosen to reach every kernel and launch path:
# compose8 + ticket, leaf folds, tree / fold_rows / walk, converge, sticky parking,
# the pipelined host path, batches, lookahead, segment fold, graph replay and PDL.
# Usage: tools/sanitize.sh OUTDIR [tool ...]   (default: memcheck racecheck synccheck initcheck)
O=${1:-gpurun_out/sanitize}
shift
TOOLS=${*:-memcheck racecheck synccheck initcheck}
mkdir -p "$O"
CS=/usr/local/cuda/bin/compute-sanitizer
# memcheck/initcheck/synccheck: every path at small sizes
K_ALL="config_small_full_parity or config_small_convergence_off or tiny_hard or tree_fanin or segment_maps_fold \
or graph_replay or sticky_parking or match_host_pipelined or match_batch or rep8_with_converge or lookahead_maps_configs \
or misaligned or edge_lengths or empty_input or alg2 or table_layouts or window or chunk_ratio_c or max_lanes \
or error_state_paper or single_kernel or alternating"
# racecheck instruments every shared access (the match loop does one per byte): small inputs only
K_RACE="config_small_full_parity and (tiny or random or keyword) or tiny_hard or tree_fanin or sticky_parking \
or rep8_with_converge or segment_maps_fold or single_kernel"
for t in $TOOLS; do
  case $t in
    racecheck) K="$K_RACE"; EXTRA="--racecheck-report all" ;;
    initcheck) K="$K_ALL"; EXTRA="" ;;
    *) K="$K_ALL"; EXTRA="" ;;
  esac
  echo "== $t" > "$O/sanitize_$t.log"
  timeout 1500 $CS --tool "$t" $EXTRA --target-processes all --print-limit 50 --error-exitcode 99 \
    python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "$K" \
    >> "$O/sanitize_$t.log" 2>&1
  echo "== rc=$?" >> "$O/sanitize_$t.log"
  tail -3 "$O/sanitize_$t.log"
done
