# r02 experiment A: L2 fetch granularity (cudaLimitMaxL2FetchGranularity) on the seam-heavy configs
set -u
mkdir -p gpurun_out
{
for c in C2 C3 C4; do
  VSTEPS=50 bash scripts/variants.sh $c "GHX_L2_FETCH=0" "GHX_L2_FETCH=32" "GHX_L2_FETCH=64" "GHX_L2_FETCH=128"
done
VSTEPS=50 bash scripts/variants.sh C2 "GHX_L2_FETCH=0|--ngrow 2,0,0" "GHX_L2_FETCH=32|--ngrow 2,0,0" "GHX_L2_FETCH=64|--ngrow 2,0,0" "GHX_L2_FETCH=0|--ngrow 0,2,2" "GHX_L2_FETCH=32|--ngrow 0,2,2"
} > gpurun_out/expA_times.txt 2>&1
{
for e in "GHX_L2_FETCH=0" "GHX_L2_FETCH=32" "GHX_L2_FETCH=64"; do
  bash scripts/ncu_metrics.sh "C2:$e" "$e" --config C2
done
} > gpurun_out/expA_ncu.txt 2>&1
cat gpurun_out/expA_times.txt gpurun_out/expA_ncu.txt
