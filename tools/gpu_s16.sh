TC2=2 timeout 120 python tools/probe_setup.py 2 2>&1 | grep "tc3\|Error\|error" | head
TC2=2 timeout 120 python tools/probe_setup.py 3 2>&1 | grep "tc3\|Error\|error" | head
