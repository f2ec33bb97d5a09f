# per-warp turning kernel for every passenger count: parity, then turning-pass times per n with
# the per-warp kernel (default) and the group kernel (QSIM_TURN_PW=0)
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_determinism.py tests/test_gpu_symmetry.py -q -m gpu -x 2>&1 | tail -2
for n in 22 23 24 25 26 27 28 29; do
  for pw in 1 0; do
    echo "== n=$n QSIM_TURN_PW=$pw"
    QSIM_TURN_PW=$pw timeout 200 python tools/pass_times.py --n $n --p 8 --reps 3 | grep "kind"
  done
done
