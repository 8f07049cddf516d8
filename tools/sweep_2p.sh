# ROUND-1 RECORD: used runtime switches (WF_SCAN_2P / WF_SCAN_TMEM) that round 2
# removed from the product library; the round-1 kernels build only as variants
# (tools/build_variants.py with -DWF_SCAN_IMPL=1|2|3), selected with WF_LIB.
mkdir -p gpurun_out
timeout 300 python tools/sweep_2p.py 64 128 256 > gpurun_out/sweep_2p.log 2>&1
for v in lead1k lead512 gap256 gap64; do WF_LIB=build/variants/lib_$v.so timeout 200 python tools/sweep_2p.py 128 >> gpurun_out/sweep_2p.log 2>&1; done
for c in 64 128 256; do WF_2P_CHUNK_TILES=$c WF_LIB=build/variants/lib_st.so timeout 100 python tools/stats_2p.py; done >> gpurun_out/sweep_2p.log 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct
WF_2P_CHUNK_TILES=128 timeout 120 ncu --metrics $M --clock-control none -k regex:two_pass -c 2 --csv python tools/profile_kernels.py c3 c4 > gpurun_out/ncu_2p_v2.csv 2>&1
cat gpurun_out/sweep_2p.log
