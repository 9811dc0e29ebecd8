for f in 0 1.4 1.5 0 1.4 1.5; do echo "capm factor $f"; VMI_CAPM_FACTOR=$f VARIANTS="base" CONFIGS="c4" bash tools/ab_run.sh 2>&1 | grep -v "^+"; done
