# same-session A/B: base library vs tools/variants/$V.so for each V in $VARS, twice
for i in 1 2; do
  timeout 300 python tools/sym_ab.py
  for v in $VARS; do GGM_LIB_PATH=tools/variants/$v.so timeout 300 python tools/sym_ab.py; done
done
