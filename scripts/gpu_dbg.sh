for cfg in "256 4 32" "2 2 64" "256 2 64" "1024 2 64" "1024 2 32" "8192 4 64" "256 2 128"; do
  timeout 60 python scripts/dbg_det.py $cfg 2>&1 | tail -1; echo "rc=$? cfg=$cfg"
done
