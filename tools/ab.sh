# A/B the assembly of several libhmx builds on the same box, alternating runs.
# usage: bash tools/ab.sh TAG lib1.so lib2.so [lib3.so ...]
tag=$1; shift
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv,noheader
for i in 1 2 3; do
  for lib in "$@"; do
    echo -n "$(basename $lib): "; HMX_LIB=$lib python tools/asm_repeat.py $tag 2 | tail -1
  done
done
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv,noheader
