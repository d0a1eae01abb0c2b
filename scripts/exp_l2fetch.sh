set -u
mkdir -p gpurun_out
for c in C3 C2; do
  VSTEPS=50 bash scripts/variants.sh $c "GHX_L2_FETCH=0" "GHX_L2_FETCH=32" "GHX_L2_FETCH=64" "GHX_L2_FETCH=128" "GHX_LD_MODE=0" "GHX_LD_MODE=1" "GHX_LD_MODE=4" "GHX_LD_MODE=3"
done > gpurun_out/exp1_times.txt 2>&1
for c in C3 C2; do
  for e in "GHX_L2_FETCH=0" "GHX_L2_FETCH=32" "GHX_LD_MODE=0" "GHX_LD_MODE=4"; do
    bash scripts/ncu_metrics.sh "$c:$e" "$e" --config $c
  done
done > gpurun_out/exp1_ncu.txt 2>&1
cat gpurun_out/exp1_times.txt gpurun_out/exp1_ncu.txt
