for p in 1 2 3; do python scripts/seg_rows_ab.py g8; PP_LIB_PATH=scripts/variants/lib_rows16.so python scripts/seg_rows_ab.py g16; done
