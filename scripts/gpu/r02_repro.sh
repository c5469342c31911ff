for k in s d c z; do
python scripts/repro_plans.py $k 3,2,1,4 45,53,23,45 45,56,23,45 24,56,45,47 0.7 1.1 2>&1 | grep -v "^$" | head -8
python scripts/repro_plans.py $k 3,1,2 56,57,63 56,57,65 58,63,56 1.0 0.0 2>&1 | head -8
done
