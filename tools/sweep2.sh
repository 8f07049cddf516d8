mkdir -p gpurun_out
( echo "== np_minb8 persist=0"; WF_LIB=build/variants/lib_np_minb8.so WF_SCAN_PERSISTENT=0 timeout 120 python tools/bench_kernels.py c3 c4 | grep -v correct
for v in p16s1 p8s3 p4s4 p8s2 p16s2 p4s6; do echo "== $v persist=1"; WF_LIB=build/variants/lib_$v.so WF_SCAN_PERSISTENT=1 timeout 120 python tools/bench_kernels.py c3 c4 ; done
echo "== trace p8s2"; WF_TRACE_TILE=8192 WF_LIB=build/variants/lib_tr_p8s2.so WF_SCAN_PERSISTENT=1 python tools/trace_scan.py
echo "== trace p4s4"; WF_TRACE_TILE=4096 WF_LIB=build/variants/lib_tr_p4s4.so WF_SCAN_PERSISTENT=1 python tools/trace_scan.py ) > gpurun_out/sweep2.log 2>&1
cat gpurun_out/sweep2.log
