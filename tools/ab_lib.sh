# A/B of two builds of libhmx.so in one GPU session (HMX_LIB selects the library):
#   bash tools/ab_lib.sh build/ab/libhmx_old.so "U32k T65k" 4
OLD=${1:-build/ab/libhmx_old.so}
CFGS=${2:-"U32k T65k"}
REPS=${3:-4}
mkdir -p gpurun_out
for cfg in $CFGS; do
  for round in 1 2; do
    echo "== $cfg old (round $round)"; HMX_LIB=$OLD python tools/asm_repeat.py $cfg $REPS 2>&1 | tail -1
    echo "== $cfg new (round $round)"; python tools/asm_repeat.py $cfg $REPS 2>&1 | tail -1
  done
done
