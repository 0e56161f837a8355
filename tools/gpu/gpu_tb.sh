AB_ARMS="default lib:tb8 lib:tb32" bash tools/gpu/gpu_ab_env.sh
