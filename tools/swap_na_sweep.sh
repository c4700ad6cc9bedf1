for na in auto 3 4 5 6 7; do
  if [ $na = auto ]; then python tools/swap_na_sweep.py; else QCF_SWAP_NA=$na python tools/swap_na_sweep.py; fi
done
