# stress the short G=8 launch (T=4096) per library build; sanitizer pass on lib_a
for i in 1 2 3 4 5 6; do for v in a b e; do PQB_TS=4096 PQB_LIB=ab/lib_$v.so timeout 60 python scripts/g8_scaling.py > gpurun_out/rp_${v}_$i.log 2>&1; echo "$v $i rc=$?"; done; done
PQB_TS=4096 PQB_LIB=ab/lib_a.so timeout 400 compute-sanitizer --tool memcheck --print-limit 5 python scripts/g8_scaling.py > gpurun_out/rp_san_a.log 2>&1; echo "san rc=$?"; tail -40 gpurun_out/rp_san_a.log | head -40
