# A/B of CSR-rows variants: bash scripts/segrows_ab.sh lib1.so lib2.so ...  (generic_probe CSR lines, 2 rounds)
for i in 1 2; do for l in "$@"; do echo "== $l"; HPAR_LIB=$l timeout 300 python scripts/generic_probe.py 2>&1 | grep "c3_fast_nest"; done; done
