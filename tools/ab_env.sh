# A/B timing of environment-selected variants on one box:
#   AB="base cta256:VMI_CTA_THREADS=256,VMI_SINGLE_MAXLOAD=0.9" CONFIGS="c2 c4" bash tools/ab_env.sh
mkdir -p gpurun_out
for spec in ${AB:-base}; do
  name=${spec%%:*}; envs=""
  case $spec in *:*) envs=$(echo ${spec#*:} | tr ',' ' ');; esac
  for c in ${CONFIGS:-c2}; do
    env $envs timeout 600 python bench.py --config $c --no-cpu-baseline --parity-sample 0 --e2e-steps 1 \
      > gpurun_out/ab_${name}_$c.json 2> gpurun_out/ab_${name}_$c.err
    python -c "import json;d=json.load(open('gpurun_out/ab_${name}_$c.json'));print('$name', d['config']['config_id'], round(d['value']), round(d['roofline']['kernel_ms'],3), d['fixups_per_step'])" || tail -3 gpurun_out/ab_${name}_$c.err
  done
done
