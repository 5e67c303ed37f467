timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_chain.py -m gpu -x -q 2>&1 | tail -3
for S in 0 1000 2000 3000 4000; do
  MACKO_CHAIN_SKEW_NS=$S timeout 300 python tools/chain_time.py --tag skew$S 2>&1 | grep -v Warn
done
