for p in 1 2; do python scripts/seg_lane_ab.py ldg; PP_LIB_PATH=scripts/variants/lib_lanestream.so python scripts/seg_lane_ab.py stream; done
