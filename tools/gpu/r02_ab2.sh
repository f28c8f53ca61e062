set -x
python tools/fwd_probe.py 4096
python tools/fwd_probe.py 11008
python tools/ab_probe.py prod
