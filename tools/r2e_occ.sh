# Plane kernel CTA shapes: more, smaller CTAs per SM at the same register budget (A/B on c3 and c5).
O=gpurun_out
bash tools/ab_r2.sh paper_1703_06256_b200/libhogb200.so build/libhog_mid128x3.so build/libhog_mid160x3.so -- c3 > $O/r2e_occ_c3.txt 2>&1
bash tools/ab_r2.sh paper_1703_06256_b200/libhogb200.so build/libhog_wide128x3.so build/libhog_wide160.so -- c5 > $O/r2e_occ_c5.txt 2>&1
