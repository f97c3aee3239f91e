for p in 1 2; do python scripts/seg_rows_ab.py base; for v in st4x48 st4x32 t3; do PP_LIB_PATH=scripts/variants/lib_$v.so python scripts/seg_rows_ab.py $v; done; done
