# Same-box A/B of library builds under tools/probes/alt/ (lib_<name>.so):
# bash tools/probes/ab_run.sh "old new" "c5ss c4ss" [rounds]
VS=${1:-"old new"}; WS=${2:-"c5ss c4ss"}; R=${3:-2}
for r in $(seq $R); do for w in $WS; do for v in $VS; do
  EBIC_B200_LIB=tools/probes/alt/lib_$v.so python tools/kernel_probe.py $w "" | sed "s/^/$v /"
done; done; done
