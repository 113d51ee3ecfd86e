python -m paper_1506_02869_b200.build > gpurun_out/build_rp.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "rollout or evaluate or replay or full_size" > gpurun_out/pytest_rp.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_rp.log
bash tools/gpu_ab2.sh rp "" "-DSMC_K2_RHOPOLY=0"
