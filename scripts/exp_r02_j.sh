# r02 experiment J: the phased exchange on DEVICE fabs (x, then y over x ghosts, then z; no edge tags)
set -u
mkdir -p gpurun_out
{
for c in C3 C2 C4; do
  VSTEPS=50 bash scripts/variants.sh $c "GHX_PHASED=0|--no-split" "GHX_PHASED=1|--no-split" "GHX_PHASED=1 GHX_BULK=1|--no-split" "GHX_PHASED=1 GHX_BULK=0|--no-split" "GHX_PHASED=1 GHX_FAB_LOCAL=0|--no-split"
done
} > gpurun_out/expJ.txt 2>&1
cat gpurun_out/expJ.txt
