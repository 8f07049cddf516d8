for rep in 1 2 3; do
for v in base nag2l3 nag2l2 nag2l4; do WF_LIB=build/variants/lib_$v.so timeout 100 python tools/bench_kernels.py c3 c4 2>&1 | sed "s#^#$v #"; done
done
for v in base nag2l3; do for rep in 1 2; do WF_LIB=build/variants/lib_$v.so python bench.py --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); c=d[\"per_kernel\"][\"c4_compact_i32\"]; print(\"bench $v\", c[\"kernel_us\"], {k:v[\"kernel_us\"] for k,v in c[\"selectivity_variants\"].items()}, d[\"per_kernel\"][\"c3_scan_i32\"][\"kernel_us\"])"; done; done
