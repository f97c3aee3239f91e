for p in 1 2 3; do python scripts/seg_rows_ab.py stcsG8; PP_LIB_PATH=scripts/variants/lib_rows0.so python scripts/seg_rows_ab.py plain; done
