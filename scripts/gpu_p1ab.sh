for l in "$@"; do BM_LIB=$PWD/$l timeout 300 python scripts/phase1_ab.py C2 C3 C4; done
