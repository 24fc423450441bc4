"""pipeplan.scheduler: the reference module also holds validate_schedule
(scheduler.py:303-452), which lives in paper_2204_10562_b200.checker here."""
from paper_2204_10562_b200.checker import validate_schedule  # noqa: F401
from paper_2204_10562_b200.model import ScheduleEvent  # noqa: F401
from paper_2204_10562_b200.scheduler import *  # noqa: F401,F403
from paper_2204_10562_b200.scheduler import ExecutionOrder, SchedulingError  # noqa: F401
