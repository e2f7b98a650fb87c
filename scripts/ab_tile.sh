for v in t1 t2 t1 t2; do cp build/variants/lib_$v.so paper_2503_21937_b200/liblobster.so; echo $v; python scripts/tile_prof.py 256 3 | tail -1; done
cp build/variants/lib_t1.so paper_2503_21937_b200/liblobster.so
