for i in 1 2; do
  echo "[new]"; timeout 300 python tools/overall_one.py
  echo "[old]"; GGM_LIB_PATH=tools/variants/old.so timeout 300 python tools/overall_one.py
done
REPS=1 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ov_new.csv python tools/overall_one.py > /dev/null 2>&1
REPS=1 GGM_LIB_PATH=tools/variants/old.so ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ov_old.csv python tools/overall_one.py > /dev/null 2>&1
