# full ncu capture of the overall rules' row-mass kernel (kSymList, mode 2) at n = 10^6
REPS=1 timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k 'regex:topk<\(int\)5, \(int\)3' -c 1 -o gpurun_out/${1:-r02_mass2} python tools/overall_one.py
