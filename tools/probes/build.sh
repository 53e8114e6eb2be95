# Builds the host-side probes (binaries are git-ignored; they travel to the GPU
# box with gpurun).  The GA probes include the reference's headers, so build
# them here, where /root/reference exists.
# usage: bash tools/probes/build.sh
set -e
cd "$(dirname "$0")/../.."
REF=/root/reference/proj/include
JSON=/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann
LINK=(-L paper_1801_03039_b200 -lebic_b200 "-Wl,-rpath,\$ORIGIN/../../paper_1801_03039_b200")
for p in ga_phase_probe build_gen_probe; do
  g++ -std=c++20 -O2 -I include -I $REF -I $JSON tools/probes/$p.cpp "${LINK[@]}" -o tools/probes/$p
done
g++ -std=c++20 -O2 -I include -I $REF -I $JSON tools/probes/build_gen_compare.cpp "${LINK[@]}" \
  -o tools/probes/build_gen_compare_dropin
g++ -std=c++20 -O2 -I $REF -I $JSON tools/probes/build_gen_compare.cpp -o tools/probes/build_gen_compare_ref
for p in launch_probe graph_launch_probe graph_update_probe launch_api_probe; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/probes/$p tools/probes/$p.cu -lcuda
done
echo "probes built"
