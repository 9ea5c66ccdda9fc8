# assembly A/B of (lib, env) variants: bash tools/ab_env.sh "U32k T65k" "lib1.so|ENV=1" "lib2.so|ENV=2" ...
cfgs=$1; shift
for c in $cfgs; do
  for i in 1 2; do
    for v in "$@"; do
      lib=${v%%|*}; envs=${v#*|}; [ "$envs" = "$v" ] && envs=""
      echo -n "$(basename $lib) [$envs] $c: "; env $envs HMX_LIB=$lib python tools/asm_repeat.py $c ${REPS:-2} | tail -1
    done
  done
done
