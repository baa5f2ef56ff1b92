timeout 900 ncu --set full --import-source on --clock-control none -k regex:k4w_multi_pair -s 3 -c 1 -o gpurun_out/r02_c18_k4wm_pair python tools/k4w_pair_profile.py 4 8 > gpurun_out/r02_c18_ncu.log 2>&1
echo done
