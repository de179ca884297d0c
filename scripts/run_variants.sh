# usage: bash scripts/run_variants.sh CONFIG STEPS lib1 lib2 ...  ("default" = in-tree libfjg.so)
# prints one summary line per variant: ms/step, last-node ms, count, checksum
cfg=$1; steps=$2; shift 2
for v in "$@"; do
  n=$(basename $v .so)
  if [ "$v" = default ]; then L=""; else L="FJG_LIB=$PWD/$v"; fi
  env $L timeout 300 python bench.py --config $cfg --steps $steps --warmup 2 --no-cpu --e2e-steps 0 \
    2>gpurun_out/v_${cfg}_$n.err | tail -1 > gpurun_out/v_${cfg}_$n.json
  python -c "import json,sys; d=json.load(open('gpurun_out/v_${cfg}_$n.json')); p=d['phases_ms']; print('$cfg', '$n', round(d['ms_per_step'],3), 'last', round(p['last_node_total'],3), d['result']['count'], d['result']['checksum'], round(d['roofline']['frac'],3))" 2>/dev/null || echo "$cfg $n FAILED $(tail -2 gpurun_out/v_${cfg}_$n.err)"
done
