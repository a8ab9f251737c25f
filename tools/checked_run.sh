#!/bin/bash
# The GPU parity suite against the bounds-checked library (tools/build_checked.py):
# any out-of-range table lookup, index or input read traps with its site, failing the
# test.  Run under gpurun; the log goes to OUTDIR.
O=${1:-gpurun_out/checked}
mkdir -p "$O"
export DFA_LIB=$PWD/paper_1210_5093_b200/libdfa_checked.so
test -f "$DFA_LIB" || { echo "missing $DFA_LIB (python tools/build_checked.py)"; exit 1; }
timeout 2400 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider > "$O/checked_pytest.log" 2>&1
echo "== rc=$?" >> "$O/checked_pytest.log"
grep -ci "illegal instruction" "$O/checked_pytest.log" | sed "s/^/trapped launches (illegal instruction): /" >> "$O/checked_pytest.log"
tail -3 "$O/checked_pytest.log"
