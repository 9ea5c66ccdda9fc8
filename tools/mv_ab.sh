# matvec A/B of several libhmx builds (alternating, 2 rounds): bash tools/mv_ab.sh lib1.so lib2.so ...
for i in 1 2; do
  for lib in "$@"; do HMX_LIB=$lib python tools/mv_ab.py 100 2>&1 | tail -1; done
done
