for dg in 2 3 4 5 6; do for rg in 10 15 25; do echo "deg $dg range $rg: $(DGB_MG_DEGREE=$dg DGB_MG_RANGE=$rg python tools/mg_timing.py cfg3 2>&1 | grep 'pressure solve mg')"; done; done
