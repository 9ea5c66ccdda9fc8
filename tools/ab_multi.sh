# A/B/C of several builds of libhmx.so in one GPU session: "cur" is the in-tree build.
#   bash tools/ab_multi.sh "cur build/ab/w10.so build/ab/w12.so" "U32k T65k" 4
LIBS=${1:-cur}
CFGS=${2:-"U32k T65k"}
REPS=${3:-4}
for cfg in $CFGS; do
  for round in 1 2; do
    for lib in $LIBS; do
      if [ "$lib" = "cur" ]; then unset HMX_LIB; else export HMX_LIB=$lib; fi
      echo "== $cfg $lib (round $round): $(python tools/asm_repeat.py $cfg $REPS 2>&1 | tail -1)"
    done
  done
done
unset HMX_LIB
