bash tools/gpu_resample_ab.sh rs4
