for cfg in "1 1024" "8 1024" "4 1024" "8 640" "4 640" "8 2048" "1 1024"; do
  set -- $cfg
  echo -n "cs=$1 min=$2: "; HMX_ACA_CS=$1 HMX_ACA_CLUSTER_MIN=$2 python tools/asm_repeat.py U32k 2 | tail -1
done
