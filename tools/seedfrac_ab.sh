for i in 1 2; do for f in 64 32 16; do
  GGM_SEED_FRAC=$f timeout 120 python tools/sym_probe.py 2>&1 | grep "n=1000000 k=100 sym=1" | sed "s/^/[frac $f] /" | cut -c1-160
done; done
