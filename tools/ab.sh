# A/B the assembly of two libhmx builds on the same box, alternating runs.
# usage: bash tools/ab.sh TAG build/ab/libhmx_old.so build/ab/libhmx_new.so
tag=$1; a=$2; b=$3
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv,noheader
for i in 1 2 3; do
  for lib in $a $b; do
    echo -n "$(basename $lib): "; HMX_LIB=$lib python tools/asm_repeat.py $tag 2 | tail -1
  done
done
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv,noheader
