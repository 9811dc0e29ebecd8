mkdir -p gpurun_out
timeout 1200 python bench.py --config c5 --steps 3 --warmup 1 > gpurun_out/r2i_c5.json 2> gpurun_out/r2i_c5.err
timeout 600 nsys --version > /dev/null 2>&1 || echo "no nsys"
