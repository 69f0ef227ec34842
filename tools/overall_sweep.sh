# overall rules at n = 10^6 (down-weighted and not) vs the lists pass's seed sample
timeout 600 python tools/overall_probe.py 2>&1 | grep -v "^$" | head -3
for f in ${FRACS:-16 4}; do echo "GGM_SEED_FRAC=$f"; GGM_SEED_FRAC=$f timeout 600 python tools/overall_probe.py 2>&1 | grep overall; done
