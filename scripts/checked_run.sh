#!/bin/bash
# The GPU suite and the randomised stress with the FJG_CHECK=1 library (device
# invariant traps at the probe / force / binding-state sites): the pool does not
# allow compute-sanitizer, so this is the memory-safety evidence we can produce.
#   bash scripts/checked_run.sh OUTDIR SECONDS
out=${1:-gpurun_out}; secs=${2:-120}
[ -f variants/checked.so ] || python scripts/build_variant.py variants/checked.so -DFJG_CHECK=1 > /dev/null
export FJG_LIB=$PWD/variants/checked.so FJG_DEBUG_SYNC=1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $out/checked_pytest.log 2>&1
echo "pytest rc=$? $(tail -1 $out/checked_pytest.log)"
timeout $((secs + 120)) python scripts/stress_parity.py 101 $secs > $out/checked_stress.log 2>&1
echo "stress rc=$? $(tail -1 $out/checked_stress.log)"
timeout $((secs + 120)) python scripts/stress_parity.py 102 $secs wide > $out/checked_stress_wide.log 2>&1
echo "stress wide rc=$? $(tail -1 $out/checked_stress_wide.log)"
