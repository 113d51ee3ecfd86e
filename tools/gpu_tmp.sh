python -m paper_1506_02869_b200.build > gpurun_out/build_ipc.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "ipc or virtual" > gpurun_out/pytest_ipc.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_ipc.log
