# Full GPU validation + evidence pass: VER=v15 bash tools/gpu_validate.sh
set -x
mkdir -p gpurun_out
V=${VER:-cur}
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$V.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$V.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$V.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_$V.json 2> gpurun_out/bench_$V.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$V.json 2> gpurun_out/bench_ref_$V.err
for c in c1 c3 c4 c5; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_${c}_$V.json 2> gpurun_out/bench_${c}_$V.err; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$V.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_l_$V.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pose_fast -s 3 -c 1 -f -o gpurun_out/k1_$V python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_f_$V.log 2>&1
ls -la gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pose_fast -s 3 -c 1 -f -o gpurun_out/k1_c4_$V python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_c4_$V.log 2>&1
