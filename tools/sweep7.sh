for m in 0 1 2 3; do
  for cfg in "8 2 4 2" "8 2 8 1" "4 2 8 2" "4 3 8 2" "8 3 4 2" "16 2 4 1" "8 4 4 1" "4 4 8 1" "8 2 8 2" "2 4 8 4"; do
    ./tools/bin/gb $m $cfg
  done
done
