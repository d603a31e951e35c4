bash tools/ab.sh old
for v in "" old; do DEBLUR_LIB_VARIANT=${v:+libdeblur_$v.so} DEBLUR_NO_GRAPHS=1 timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:k_cols_tm --launch-skip 4 -c 2 python tools/prof_step.py 4 3 2>&1 | grep -E "k_cols_tm|dram__|gpu__time" | head -8; done
