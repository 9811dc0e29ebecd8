# ncu evidence for several configs (each plain run first, then one ncu capture of K1)
#   CFGS="c4:16384 c3:65536" TAG=r02_v0 bash tools/gpu_prof.sh
mkdir -p gpurun_out
for spec in ${CFGS:-c2:65536}; do
  c=${spec%%:*}; P=${spec#*:}
  cmd="python bench.py --config $c --poses $P --steps 1 --warmup 3 --no-cpu-baseline --parity-sample 0 --e2e-steps 1"
  if [ $c = c3 ]; then cmd="$cmd"; fi
  timeout 600 $cmd > gpurun_out/${TAG}_${c}_plain.json 2> gpurun_out/${TAG}_${c}_plain.err && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pose_fast -s 3 -c 1 -f \
      -o gpurun_out/${TAG}_${c} $cmd > gpurun_out/${TAG}_${c}_ncu.log 2>&1
  echo "$c rc=$?"
done
