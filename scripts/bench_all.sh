# Refresh every config's bench line: bash scripts/bench_all.sh TAG
tag=${1:-r01}
for cfg in ${CFGS:-chain triangle star clique4 scale_triangle scale_path5}; do
  case $cfg in scale_*) a="--steps 3 --warmup 3 --e2e-steps 0 --no-cpu";; clique4) a="--steps 5 --warmup 3";; *) a="";; esac
  timeout 1200 python bench.py --config $cfg $a > gpurun_out/${tag}_bench_$cfg.json 2> gpurun_out/${tag}_bench_$cfg.err
  tail -1 gpurun_out/${tag}_bench_$cfg.json | cut -c1-200
done
