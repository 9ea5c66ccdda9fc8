HMX_ACA_TC=1 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for lib in tc2 tc3; do
echo -n "$lib base U131k: "; HMX_LIB=build/ab/libhmx_$lib.so python tools/asm_repeat.py U131k 2 | tail -1
echo -n "$lib tc U131k:   "; HMX_LIB=build/ab/libhmx_$lib.so HMX_ACA_TC=1 python tools/asm_repeat.py U131k 2 | tail -1
echo -n "$lib tc T65k:   "; HMX_LIB=build/ab/libhmx_$lib.so HMX_ACA_TC=1 python tools/asm_repeat.py T65k 2 | tail -1
echo -n "$lib tc U32k:   "; HMX_LIB=build/ab/libhmx_$lib.so HMX_ACA_TC=1 python tools/asm_repeat.py U32k 2 | tail -1
done
