# Full EBIC runs (generate -> GA run -> finalize -> write JSON) through the
# reference's own API: the pure reference build (CPU, all host threads) vs the
# same driver compiled against the shadow headers (B200 drop-in).  Prints the
# phase timings of both and whether the JSON outputs are byte-identical.
# Also replays recorded top-rank streams through both TopRankList builds.
# usage (GPU box): bash tools/ga_run_compare.sh
mkdir -p gpurun_out
out=gpurun_out/ga_compare.log
: > $out
T=$(nproc)
run_pair() {  # name, args...
  local name=$1; shift
  echo "== $name ($*)" >> $out
  ./oracle/_ref/ebic_ref_run "$@" threads=$T out=/tmp/ga_ref_$name.json 2>> $out
  ./oracle/_ref/ebic_dropin_run "$@" threads=$T out=/tmp/ga_dropin_$name.json 2>> $out
  if cmp -s /tmp/ga_ref_$name.json /tmp/ga_dropin_$name.json; then echo "json identical" >> $out; else echo "JSON DIFFERS" >> $out; fi
}
# BASELINE.json configs 0 and 3 at their stated iteration counts.
run_pair c1 rows=500 cols=100 blocks=50x10,50x10,50x10 seed=1 population=600 iterations=1000 rng_seed=42 epsilon=1e-9 overlap_threshold=0.5 threshold=none
# C4 shape with every top-rank entry written (threshold none): ~10^6 expanded rows in the output.
run_pair c4_all rows=20000 cols=500 blocks=600x20,600x20,600x20,600x20,600x20 seed=2026 population=600 iterations=200 rng_seed=1 epsilon=1e-9 threshold=none
run_pair c4 rows=20000 cols=500 blocks=600x20,600x20,600x20,600x20,600x20 seed=2026 population=600 iterations=5000 rng_seed=1 epsilon=1e-9
cat $out
