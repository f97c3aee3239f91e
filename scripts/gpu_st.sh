for p in 1 2 3; do python scripts/count_ab.py ncw8; for v in ncw16 ncw12 ncw4s6; do PP_LIB_PATH=scripts/variants/lib_$v.so python scripts/count_ab.py $v; done; done
