# Solve time per speculative slot count (EVD_SPEC_K) and CTA size on cfg 1-2.
for b in 384 512; do for k in 1 2 3 4; do echo "block $b spec $k"; EVD_SOLVE_BLOCK=$b EVD_SPEC_K=$k python tools/time_solve.py 1 2; done; done
