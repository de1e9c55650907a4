export PATH=/usr/local/cuda/bin:$PATH
CONFIGS="${CONFIGS:-5a 2 1 3a 3b 3c 4a 4b 5a-f32 5b}" bash tools/refresh_profiles.sh
