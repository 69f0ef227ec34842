# Same-session A/B: per-row re-evaluation cuts forced (GGM_REC_CUT=1) vs the default (cuts only
# for candidate-heavy pools), C4 and C5 sizes.
set -u
for i in 1 2 3; do
  timeout 300 python tools/sym_ab.py
  GGM_REC_CUT=1 TAG=reccut timeout 300 python tools/sym_ab.py
done
