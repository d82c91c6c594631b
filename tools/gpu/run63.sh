AB_ATTR="sched_priorities=False,node_priority=False|sched_priorities=True,node_priority=False|sched_priorities=True,node_priority=True" timeout 600 python tools/skip_frame.py C3 2>&1 | tail -6
