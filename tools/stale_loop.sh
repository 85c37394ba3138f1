for mode in "" "RN_BN_FIN_INLINE=1" "RN_PDL=0"; do
  fails=0
  for i in 1 2 3 4 5 6; do
    env $mode timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "stale" > /tmp/o.txt 2>&1 || fails=$((fails+1))
  done
  echo "mode [$mode] fails $fails/6"
done
grep -E "^E " /tmp/o.txt | head
