# assembly A/B of several libhmx builds over several configs (rep-1 totals)
# usage: bash tools/ab_cfg.sh "U32k T65k" lib1.so lib2.so ...
cfgs=$1; shift
for c in $cfgs; do
  for i in 1 2; do
    for lib in "$@"; do
      echo -n "$(basename $lib) $c: "; HMX_LIB=$lib python tools/asm_repeat.py $c 2 | tail -1
    done
  done
done
