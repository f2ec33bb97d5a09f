# split-run parameter a (QSIM_RUNSPLIT) with the final kernels: per-pass means at n = 30, p = 8
for a in 4 2 3 5 6 0 4; do
  echo "== QSIM_RUNSPLIT=$a"
  QSIM_RUNSPLIT=$a timeout 200 python tools/pass_times.py --n 30 --p 8 --reps 3 | grep "kind"
done
