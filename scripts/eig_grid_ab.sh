O=gpurun_out
for g in head 32 148 head; do cp abtest/libskp_$g.so paper_2605_09755_b200/libskp.so; python scripts/eig_time.py 520 1050 | sed "s/^/grid $g /"; done 2>&1 | tee $O/eig_grid_ab.txt
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv
