# SCT lane-kernel iteration: parity tests of the lane / fast kernels, then throughput of the
# warp, lane and fast kernels at k=10, n=400 (bigram and trigram) -- scripts/prof_sct.py
timeout 900 python -m pytest tests/test_gpu_sct_lane.py -x -q 2>&1 | tail -3
for W in ${WS:-16384 65536 131072}; do
for o in 2 3; do for kern in warp lane fast; do echo -n "W=$W "; timeout 300 python scripts/prof_sct.py --order $o --kernel $kern --workers $W --climbings 2000 --reps 2 | tail -1; done; done
done
