for dl in 1 0; do AIRG_DEVLOOP=$dl python tools/gm_probe.py --fast 1; done
AIRG_DEVLOOP=1 python tools/gm_probe.py --fast 0
