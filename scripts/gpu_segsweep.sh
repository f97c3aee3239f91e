#!/bin/bash
for p in ldg tma; do PP_SEG_PATH=$p timeout 300 python scripts/seg_sweep.py; done
