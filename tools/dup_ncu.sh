for v in old duprow dupcol dupgram; do
  HMX_LIB=build/ab/libhmx_$v.so ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_bytes.sum -k regex:aca_kernel -c 2 python tools/ncu_target.py U32k 1 2>&1 | grep -E "aca_kernel|duration|bytes" | sed "s/^/$v /"
done
