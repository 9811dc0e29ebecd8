# A/B timing of variant builds: VARIANTS="base x y" CONFIGS="c2 c4" bash tools/ab_run.sh
mkdir -p gpurun_out
for v in ${VARIANTS:-base}; do
  if [ $v = base ]; then L=""; else L="abvar/$v/libvmi.so"; fi
  for c in ${CONFIGS:-c2}; do
    VMI_LIB=$L python bench.py --config $c --no-cpu-baseline --parity-sample 0 --e2e-steps 1 > gpurun_out/ab_${v}_$c.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/ab_${v}_$c.json'));print('$v', d['config']['config_id'], round(d['value']), round(d['roofline']['kernel_ms'],3), d['fixups_per_step'])"
  done
done
