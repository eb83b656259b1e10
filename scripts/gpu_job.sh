A_LIB=$PWD/paper_2304_08662_b200/_lib/libxdrop_b200_A.so bash scripts/ab_run.sh "--config 5 --scale 1.0" "--config 4 --scale 1.0" "--config 5 --scale 0.5 --x 40"
