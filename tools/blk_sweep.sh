# Solve time per CTA size (EVD_SOLVE_BLOCK) on the large windows (cfg 3, 5).
for b in 512 768 1024; do echo "block $b"; EVD_SOLVE_BLOCK=$b python tools/time_solve.py ${CFGS:-3 5}; done
