# Full GPU validation + evidence pass: VER=r02_vX bash tools/gpu_validate.sh
mkdir -p gpurun_out
V=${VER:-cur}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$V.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$V.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$V.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$V.log
timeout 900 python bench.py > gpurun_out/bench_c2_$V.json 2> gpurun_out/bench_c2_$V.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$V.json 2> gpurun_out/bench_ref_$V.err
for c in c1 c1v c3 c4; do timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_${c}_$V.json 2> gpurun_out/bench_${c}_$V.err; done
timeout 1200 python bench.py --config c5 --steps 3 --warmup 1 > gpurun_out/bench_c5_$V.json 2> gpurun_out/bench_c5_$V.err
timeout 900 python bench.py --config c5 --impl reference --steps 1 --warmup 0 > gpurun_out/bench_c5ref_$V.json 2> gpurun_out/bench_c5ref_$V.err
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --parity-sample 0 --e2e-steps 1 > gpurun_out/ncu_plain_$V.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$V.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --parity-sample 0 --e2e-steps 1 > gpurun_out/ncu_l_$V.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pose_fast -s 3 -c 1 -f -o gpurun_out/k1_c2_$V python bench.py --steps 1 --warmup 3 --no-cpu-baseline --parity-sample 0 --e2e-steps 1 > gpurun_out/ncu_f_$V.log 2>&1
for spec in c1:1 c1v:1 c3:1 c4:65536; do
  c=${spec%%:*}; P=${spec#*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pose_fast -s 3 -c 1 -f -o gpurun_out/k1_${c}_$V python bench.py --config $c --poses $P --steps 1 --warmup 3 --no-cpu-baseline --parity-sample 0 --e2e-steps 1 > gpurun_out/ncu_${c}_$V.log 2>&1
done
# summaries on the box (gpurun_out comes back only under 64 MiB): keep C2's report
for c in c2 c1 c1v c3 c4; do
  [ -f gpurun_out/k1_${c}_$V.ncu-rep ] && python tools/ncu_summary.py full gpurun_out/k1_${c}_$V.ncu-rep gpurun_out/k1_${c}_${V}_full.json > /dev/null 2>&1
  [ $c != c2 ] && rm -f gpurun_out/k1_${c}_$V.ncu-rep
done
[ -f gpurun_out/launches_$V.csv ] && python tools/ncu_summary.py launches gpurun_out/launches_$V.csv gpurun_out/launches_${V}.json > /dev/null 2>&1
ls -la gpurun_out
