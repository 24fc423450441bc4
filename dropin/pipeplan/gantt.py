"""pipeplan.gantt: the reference's own module (out of scope here),
executed as a submodule of the drop-in so it runs on the drop-in's planner."""
from pipeplan import _exec_reference

_exec_reference("gantt", globals())
