set -x
mkdir -p gpurun_out
for v in default sbuf3 default sbuf3; do
  if [ $v = default ]; then unset HARAG_LIB; else export HARAG_LIB=build/variants/$v/libharag.so; fi
  echo "$v $(timeout 120 python tools/prof_attend.py 8 2>&1 | tail -1)"
done > gpurun_out/attend_variants2.txt 2>&1; cat gpurun_out/attend_variants2.txt
unset HARAG_LIB
for v in trace sbuf3_trace; do
HARAG_LIB=build/variants/$v/libharag.so timeout 300 python tools/prof_attend.py 1 > gpurun_out/trace_$v.txt 2>&1
python tools/trace_attend.py gpurun_out/trace_$v.txt > gpurun_out/trace_${v}_summary.txt 2>&1; cat gpurun_out/trace_${v}_summary.txt
done
