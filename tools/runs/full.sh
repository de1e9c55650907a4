export PATH=/usr/local/cuda/bin:$PATH
CONFIGS="5a 5a-f32 4b 4a 3c 3a 5b" KEEP="none" bash tools/refresh_full.sh
