# NEXT-row measurements (one B200): QSDS / <sigma^z> / Hadamard at n = 30, enumeration N = 30..40
python tools/next_bench.py --qubits 30 --steps 16 2>&1 | grep "{"
python tools/tfe_bench.py --qubits 30 32 34 36 38 40 2>&1 | grep "{"
