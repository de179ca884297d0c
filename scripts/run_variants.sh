# usage: bash scripts/run_variants.sh CONFIG STEPS lib1 lib2 ...  ("default" = in-tree libfjg.so)
cfg=$1; steps=$2; shift 2
for v in "$@"; do
  n=$(basename $v .so)
  if [ "$v" = default ]; then L=""; else L="FJG_LIB=$PWD/$v"; fi
  env $L timeout 600 python bench.py --config $cfg --steps $steps --warmup 3 --no-cpu --e2e-steps 0 2>gpurun_out/v_${cfg}_$n.err | tail -1 > gpurun_out/v_${cfg}_$n.json
done
