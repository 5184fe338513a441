export PYTHONUNBUFFERED=1
for mn in 00 10 01 11; do echo "== debug mn=$mn"; timeout 300 python tools/unit_stats.py --what debug --mn $mn 2>&1 | grep -E "cycles per|wait full"; done
echo "== stats"; timeout 300 python tools/unit_stats.py --what stats --chunk 2 2>&1 | grep -E "cycles per|wait full|wait TMEM|producer"
