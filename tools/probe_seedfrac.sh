# overall-rules phase probe at n = 1e6 (default seed fraction unless GGM_SEED_FRAC is set)
GGM_DEBUG_OVERALL=1 timeout 300 python tools/overall_probe.py 2>&1 | grep -E "overall|top-32" | uniq
