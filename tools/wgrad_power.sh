# Clocks / power per kernel phase at the C3 wgrad shape (run on a GPU box).
# usage: bash tools/wgrad_power.sh [h f G secs phases]
set -e
cd "$(dirname "$0")/.."
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_2303_06318_b200/csrc \
  tools/wgrad_power.cu -o tools/wgrad_power -L paper_2303_06318_b200 -lted_b200 \
  -Xlinker -rpath -Xlinker '$ORIGIN/../paper_2303_06318_b200' 2>/dev/null || true
mkdir -p gpurun_out
nvidia-smi --query-gpu=timestamp,clocks.sm,power.draw,clocks_event_reasons.active --format=csv,noheader -lms 50 > gpurun_out/wp_clocks.csv &
SMI=$!
sleep 1
./tools/wgrad_power "$@" > gpurun_out/wp_phases.txt
kill $SMI
python tools/wgrad_power_summary.py gpurun_out/wp_phases.txt gpurun_out/wp_clocks.csv
