# A/B several builds of libegsolve.so (EGSOLVE_LIB) with scripts/kernel_ab.py
for L in "$@"; do
  echo "### $L"
  EGSOLVE_LIB=$L python scripts/kernel_ab.py --rounds ${ROUNDS:-3} 2>&1 | grep -vE "scale|start|finalize"
done
