# A/B of the tensor-core ACA (HMX_ACA_TC=1) against the default on one box
lib=${1:-paper_1706_09384_b200/libhmx.so}
for i in 1 2; do
  echo -n "base: "; HMX_LIB=$lib python tools/asm_repeat.py U32k 2 | tail -1
  echo -n "tc:   "; HMX_LIB=$lib HMX_ACA_TC=1 python tools/asm_repeat.py U32k 2 | tail -1
done
echo -n "base T65k: "; HMX_LIB=$lib python tools/asm_repeat.py T65k 2 | tail -1
echo -n "tc T65k:   "; HMX_LIB=$lib HMX_ACA_TC=1 python tools/asm_repeat.py T65k 2 | tail -1
