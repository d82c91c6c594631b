# A/B of Simulation attributes on the C3 frame: bash tools/gpu/ab.sh "attr=v1|attr=v2" [config]
AB_ATTR="$1" timeout 600 python tools/skip_frame.py ${2:-C3} 2>&1 | tail -8
