# ROUND-1 RECORD: used runtime switches (WF_SCAN_2P / WF_SCAN_TMEM) that round 2
# removed from the product library; the round-1 kernels build only as variants
# (tools/build_variants.py with -DWF_SCAN_IMPL=1|2|3), selected with WF_LIB.
mkdir -p gpurun_out
for v in st_l1 st_l2; do for c in 256 512; do WF_2P_CHUNK_TILES=$c WF_LIB=build/variants/lib_$v.so timeout 100 python tools/stats_2p.py; done; done > gpurun_out/stats_2p.log 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct
for c in 128 256 512; do WF_2P_CHUNK_TILES=$c timeout 120 ncu --metrics $M --clock-control none -k regex:two_pass -c 2 --csv python tools/profile_kernels.py c3 c4 > gpurun_out/ncu_2p_l1_$c.csv 2>&1; done
for c in 128 256; do WF_2P_CHUNK_TILES=$c WF_LIB=build/variants/lib_lag2.so timeout 120 ncu --metrics $M --clock-control none -k regex:two_pass -c 2 --csv python tools/profile_kernels.py c3 c4 > gpurun_out/ncu_2p_l2_$c.csv 2>&1; done
cat gpurun_out/stats_2p.log
