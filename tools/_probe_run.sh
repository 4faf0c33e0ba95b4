for i in 1 2; do
for c in 2 4 5; do
  echo "cfg$c: $(python tools/prof_half_step.py --config $c --reps 10 --kernel tc 2>&1 | tail -1)"
done
done
