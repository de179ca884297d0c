# §5.3 backend ladder on the device: bash scripts/ablation.sh TAG
tag=${1:-r01}
for cfg in ${CFGS:-chain triangle star clique4}; do
  for b in colt slt simple; do
    case $cfg in clique4) a="--steps 3 --warmup 2";; *) a="--steps 10 --warmup 3";; esac
    timeout 900 python bench.py --config $cfg --backend $b $a --no-cpu --e2e-steps 0 2> gpurun_out/${tag}_abl_${cfg}_$b.err | tail -1 > gpurun_out/${tag}_abl_${cfg}_$b.json
  done
done
