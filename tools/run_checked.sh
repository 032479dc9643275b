#!/bin/bash
# Checked-build tier (the compute-sanitizer substitute: sanitizer runs are
# closed on this GPU pool, profiles/r02_sanitizer_pool_closed.txt). The
# library built with -DAMUN_CHECKS (python -c "import __graft_entry__ as g;
# g.build(extra=['-DAMUN_CHECKS'], lib='abl/libamun_checked.so')"): every
# mbarrier wait traps with its barrier after ~2 s instead of hanging (the
# pipeline / tail protocols), and bounds / invariant asserts (AMUN_DCHECK)
# trap on partial-record slots, merge record ranges, compaction ranks and
# offsets. Runs every kernel's small cases (with bit-determinism repeats)
# and the whole GPU test suite against that library.
# Usage (GPU box): bash tools/run_checked.sh [outdir]
out=${1:-gpurun_out/checked}
mkdir -p "$out"
export AMUN_LIB=$PWD/abl/libamun_checked.so
python -c "import paper_1805_09863_b200 as m; print('loaded', m.lib_path)" > "$out/lib.txt" 2>&1
timeout 900 python tools/sanitize_cases.py > "$out/cases.log" 2>&1
echo "cases rc=$?" | tee -a "$out/summary.txt"
timeout 2400 python -m pytest tests -m gpu -q > "$out/pytest.log" 2>&1
echo "pytest rc=$?" | tee -a "$out/summary.txt"
tail -3 "$out/pytest.log" >> "$out/summary.txt"
