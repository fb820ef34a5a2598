set -u
timeout 300 python tools/sanitize_cases.py; echo "cases rc=$?"
SAN_TIMEOUT=900 bash tools/sanitize.sh r3m memcheck synccheck racecheck
