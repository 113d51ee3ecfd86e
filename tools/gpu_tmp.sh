bash tools/gpu_ab2.sh qrow "" "-DSMC_K2_MINB=5 -DSMC_K2_QROW_SMEM=1" "-DSMC_K2_QROW_SMEM=1"
