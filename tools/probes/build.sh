# Builds the host-side probes (binaries are git-ignored; they travel to the GPU
# box with gpurun).  The GA probes include the reference's headers, so build
# them here, where /root/reference exists.
# usage: bash tools/probes/build.sh
set -e
cd "$(dirname "$0")/../.."
REF=/root/reference/proj/include
JSON=/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann
LINK=(-L paper_1801_03039_b200 -lebic_b200 "-Wl,-rpath,\$ORIGIN/../../paper_1801_03039_b200")
g++ -std=c++20 -O2 -I include -I $REF -I $JSON tools/probes/ga_phase_probe.cpp "${LINK[@]}" -o tools/probes/ga_phase_probe
g++ -std=c++20 -O2 -I include -I $REF -I $JSON tools/probes/build_gen_compare.cpp "${LINK[@]}" \
  -o tools/probes/build_gen_compare_dropin
g++ -std=c++20 -O2 -I $REF -I $JSON tools/probes/build_gen_compare.cpp -o tools/probes/build_gen_compare_ref
g++ -std=c++17 -O2 tools/probes/startup_probe.cpp -ldl -o tools/probes/startup_probe
for p in graph_update_probe launch_floor_probe gather_probe param_probe launch_cost_probe; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/probes/$p tools/probes/$p.cu -lcuda
done
echo "probes built"
