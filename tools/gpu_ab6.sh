for f in 2.5 2.0 2.2 2.5 2.0 2.2; do echo "cap factor $f"; VMI_CAP_FACTOR=$f VARIANTS="base" CONFIGS="c2 c1" bash tools/ab_run.sh 2>&1 | grep -v "^+"; done
